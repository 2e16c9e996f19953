#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for pdl in 1 0; do echo "== OWQ_CC_PDL=$pdl"; for a in "4096 4096 3 0 5" "4096 4096 4 128 4" "11008 4096 4 128 1" "12288 12288 3 0 15"; do OWQ_CC_PDL=$pdl OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/cc_trace.py $a 8 | head -1; done; done) 2>&1 | tee gpurun_out/cc6.txt
