#!/bin/bash
# batched f16 kernel after the z prefetch + one-wave plan: tests + timing
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_batch_f16.py -x -q > gpurun_out/sb2_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sb2_tests.txt
for a in "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 4" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16" "12288 12288 4 128 15 8" "4096 4096 4 128 4 8" "49152 12288 3 0 3 8"; do
  timeout 120 python tools/prof_batch.py $a 24
done 2>&1 | tee gpurun_out/sb2_time.txt
