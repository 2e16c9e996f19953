#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch_f16.py -q -x -p no:cacheprovider > gpurun_out/sb1.txt 2>&1; echo "batch_f16 rc=$?"; tail -30 gpurun_out/sb1.txt
for s in "12288 12288 3 0 15 2" "12288 12288 3 0 15 4" "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "12288 12288 3 0 15 32" \
         "11008 4096 4 128 1 4" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16" "4096 4096 4 128 4 8" "12288 12288 4 128 15 8" \
         "49152 12288 3 0 3 8"; do timeout 120 python tools/prof_batch.py $s; done 2>&1 | tee gpurun_out/sb_time.txt
