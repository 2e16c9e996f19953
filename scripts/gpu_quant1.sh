#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantizer.py -q -x -p no:cacheprovider > gpurun_out/quant1.txt 2>&1; echo "quant rc=$?"; tail -30 gpurun_out/quant1.txt
for s in "768 768 3 8 0" "4096 4096 3 5 0" "4096 4096 4 4 128" "12288 12288 3 15 0"; do timeout 300 python tools/quant_time.py $s; done 2>&1 | tee gpurun_out/quant_time.txt
