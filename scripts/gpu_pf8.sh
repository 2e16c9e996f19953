#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -3
for k in 15 0; do OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 200 python tools/pf_trace.py 12288 12288 2048 $k 2>&1 | tail -9; done | tee gpurun_out/pf8_trace.txt
for a in "12288 12288 2048" "12288 12288 256" "49152 12288 1024" "4096 4096 2048"; do timeout 120 python tools/prof_prefill.py $a 4; done 2>&1 | tee gpurun_out/pf8_time.txt
