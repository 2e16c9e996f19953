#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
export OWQ_LIB=paper_2306_02272_b200/_ab/exp.so
(echo "== 12288^2 B8"; timeout 120 python tools/sb_trace.py 12288 12288 3 0 15 8 | tail -16
echo "== llama up B8"; timeout 120 python tools/sb_trace.py 11008 4096 4 128 1 8 | tail -16) 2>&1 | tee gpurun_out/sb6_trace.txt
