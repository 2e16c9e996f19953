#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -2
for rb in 1 2; do OWQ_PF_RB=$rb OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -1; done
(for rb in 1 2; do echo "== RB=$rb"; for a in "12288 12288 2048" "12288 12288 256" "12288 12288 512" "49152 12288 1024" "4096 4096 2048" "4096 4096 256" "11008 4096 128"; do OWQ_PF_RB=$rb OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_prefill.py $a 4; done; done
echo "== product"; for a in "12288 12288 2048" "12288 12288 256" "12288 12288 512" "49152 12288 1024" "4096 4096 2048" "4096 4096 256" "11008 4096 128"; do timeout 120 python tools/prof_prefill.py $a 4; done) 2>&1 | tee gpurun_out/pf10_time.txt
