#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_guards.py tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -q -x -p no:cacheprovider -k "not cc" > gpurun_out/w2.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/w2.txt
for s in "12288 12288" "49152 12288"; do for k in 0 15 76 153; do timeout 120 python tools/prof_gemv.py $s 3 0 $k 1 24 3; done; done 2>&1 | tee gpurun_out/ksweep2.txt
