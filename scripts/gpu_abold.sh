#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
ls -la paper_2306_02272_b200/_ab/old.so
(for B in 1 2 4 8 16; do
  echo -n "old "; OWQ_LIB=paper_2306_02272_b200/_ab/old.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "new "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done) 2>&1 | tee gpurun_out/abold.txt
