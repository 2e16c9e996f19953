#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for sk in 15 20 25 30; do echo -n "skew $sk "; OWQ_SKEW=$sk OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 40; done
 for sk in 0 5 8 10 13 16; do for a in "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12"; do echo -n "skew $sk "; OWQ_SKEW=$sk OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $a; done; done) 2>&1 | tee gpurun_out/skew4.txt
