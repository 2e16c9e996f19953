#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for r in 0 3 6 12 24; do echo "== reserve ${r} KB"; for a in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12"; do OWQ_SMEM_RESERVE=$r OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $a; done; done) 2>&1 | tee gpurun_out/reserve.txt
