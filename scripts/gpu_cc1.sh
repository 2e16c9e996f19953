#!/bin/bash
# CUDA-core path: parity (both layouts), then timing of both layouts at the bench shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cc" > gpurun_out/cc_par1.txt 2>&1; echo "cc parity rc=$?"; tail -15 gpurun_out/cc_par1.txt
for shape in "12288 12288 3 0 15 1 40 4" "49152 12288 3 0 3 1 12 4" "12288 49152 3 0 15 1 12 4" "4096 4096 3 0 5 1 40 4" "12288 12288 4 128 15 1 40 4" "12288 12288 3 0 15 2 40 4" "12288 12288 3 0 15 4 40 4"; do timeout 120 python tools/prof_gemv.py $shape; done 2>&1 | tee gpurun_out/cc_table1.txt
