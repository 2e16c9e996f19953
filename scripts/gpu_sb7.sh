#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
export OWQ_LIB=paper_2306_02272_b200/_ab/exp.so
for sk in 0 16 15 31 47 63; do
  echo "== skip $sk"; OWQ_SB_SKIP=$sk timeout 120 python tools/sb_trace.py 12288 12288 3 0 15 8 | sed -n '2,12p;60,64p;/graph:/p'
done 2>&1 | tee gpurun_out/sb7_trace.txt
