#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
(for B in 1 4 8 16; do
  echo -n "old(746ebfd) "; OWQ_LIB=paper_2306_02272_b200/_ab/old.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "summer-low   "; OWQ_LIB=paper_2306_02272_b200/_ab/sl.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "current      "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done
for L in old sl; do echo -n "$L fc1 "; OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 8; done; echo -n "current fc1 "; timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 8) 2>&1 | tee gpurun_out/abold2.txt
