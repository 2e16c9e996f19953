#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for sk in 0 10 20 30; do echo "== OWQ_CC_SKEW=$sk"; for a in "4096 4096 3 0 5 1 40 4" "4096 4096 4 128 4 1 40 4" "11008 4096 4 128 1 1 40 4" "4096 11008 4 128 4 1 40 4" "12288 12288 4 128 15 1 20 4"; do OWQ_CC_SKEW=$sk OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $a; done; done) 2>&1 | tee gpurun_out/ccskew.txt
OWQ_CC_SKEW=30 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 120 2>&1 | tail -2
