#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
(for B in 2 4 8 16; do for sk in auto 0; do
  if [ "$sk" = auto ]; then unset OWQ_SKEW; else export OWQ_SKEW=$sk; fi
  echo -n "skew $sk "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "skew $sk "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 $B 8
done; done) 2>&1 | tee gpurun_out/skew6.txt
