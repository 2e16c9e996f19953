#!/bin/bash
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for r in 1 2; do
  shape="49152 12288 3 0 3 1 12"
  echo -n "A        "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape
  echo -n "B        "; timeout 120 python tools/prof_gemv.py $shape
  echo -n "B pdl0   "; OWQ_PDL=0 timeout 120 python tools/prof_gemv.py $shape
  echo -n "B seq    "; OWQ_EXP=4 timeout 120 python tools/prof_gemv.py $shape
  echo -n "B both   "; OWQ_EXP=4 OWQ_PDL=0 timeout 120 python tools/prof_gemv.py $shape
done
