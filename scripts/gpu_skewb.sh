#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
(for B in 1 2 3 4 8; do
  echo -n "maxb1  "; OWQ_LIB=paper_2306_02272_b200/_ab/sk1.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "maxb2  "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "maxb16 "; OWQ_LIB=paper_2306_02272_b200/_ab/sk16.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done) 2>&1 | tee gpurun_out/skewb.txt
