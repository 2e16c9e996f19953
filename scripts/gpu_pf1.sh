#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x -p no:cacheprovider > gpurun_out/pf1.txt 2>&1; echo "prefill rc=$?"; tail -30 gpurun_out/pf1.txt
for s in "12288 12288 2048" "12288 12288 256" "49152 12288 1024" "4096 4096 2048"; do timeout 120 python tools/prof_prefill.py $s; done 2>&1 | tee gpurun_out/pf_time.txt
