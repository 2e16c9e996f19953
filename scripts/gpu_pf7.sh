#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
for k in 15 0; do OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 200 python tools/pf_trace.py 12288 12288 2048 $k 2>&1 | tail -9; done | tee gpurun_out/pf7_trace.txt
