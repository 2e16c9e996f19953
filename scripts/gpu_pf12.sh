#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
for w in 0 1; do OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 200 python tools/pf_trace.py 4096 4096 256 5 $w 2>&1 | tail -12; done | tee gpurun_out/pf12_trace.txt
