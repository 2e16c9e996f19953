#!/bin/bash
# A/B on one box: A = paper_2306_02272_b200/_ab/libowq_a.so, B = in-tree libowq.so
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for r in 1 2; do
  for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "4096 4096 3 0 5 1 40"; do
    echo -n "A "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape
    echo -n "B "; timeout 120 python tools/prof_gemv.py $shape
  done
done
