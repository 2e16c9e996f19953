#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_guards.py -q --timeout 300 2>&1 | grep -E "^E |passed|failed" | head
(for a in "12288 12288 2048" "49152 12288 1024" "12288 49152 512" "4096 4096 2048" "12288 12288 256" "4096 4096 256" "4096 11008 128" "11008 4096 128"; do timeout 120 python tools/prof_prefill.py $a 4 1; done) 2>&1 | tee gpurun_out/pf15_time.txt
