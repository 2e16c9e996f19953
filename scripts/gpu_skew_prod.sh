#!/bin/bash
# product-vs-product: span skew at every B (product) vs only at B = 1 (_ab/skewb1.so)
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
(for rep in 1 2; do for B in 2 4 8 16; do
  echo -n "all-B  "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "B1-only "; OWQ_LIB=paper_2306_02272_b200/_ab/skewb1.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done; done
for B in 4 8; do
  echo -n "all-B  "; timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 $B 8
  echo -n "B1-only "; OWQ_LIB=paper_2306_02272_b200/_ab/skewb1.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 $B 8
done) 2>&1 | tee gpurun_out/skew_prod.txt
