#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_CC_MINB=2 --out paper_2306_02272_b200/_ab/exp_m2.so > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_CC_MINB=2 -D OWQ_CC_NW=4 --out paper_2306_02272_b200/_ab/exp_m2w4.so > /dev/null
(for L in exp exp_m2 exp_m2w4; do echo "== $L"; for a in "4096 4096 3 0 5" "4096 4096 4 128 4" "11008 4096 4 128 1" "4096 11008 4 128 4" "12288 12288 3 0 15"; do OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/cc_trace.py $a 8 2>/dev/null | sed -n '1p;4,6p'; done; done) 2>&1 | tee gpurun_out/cc7.txt
