#!/bin/bash
# batched f16 + prefill kernels after the async x-tile arrivals and per-row drains
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_batch_f16.py tests/test_gpu_prefill.py -x -q > gpurun_out/sb3_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sb3_tests.txt
for a in "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 4" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16" "12288 12288 4 128 15 8" "4096 4096 4 128 4 8" "49152 12288 3 0 3 8"; do
  timeout 120 python tools/prof_batch.py $a 24
done 2>&1 | tee gpurun_out/sb3_time.txt
for a in "12288 12288 2048" "12288 12288 256" "49152 12288 1024" "4096 4096 2048"; do timeout 120 python tools/prof_prefill.py $a 4; done 2>&1 | tee gpurun_out/pf3_time.txt
