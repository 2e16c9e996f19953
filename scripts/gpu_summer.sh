#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for B in 1 4 8 16; do for e in 0 7; do echo -n "exp $e "; OWQ_EXP=$e OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24; done; done
 for e in 0 7; do echo -n "exp $e "; OWQ_EXP=$e OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 8; done) 2>&1 | tee gpurun_out/summer.txt
OWQ_EXP=7 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small_batch_parity" --timeout 120 2>&1 | tail -1
