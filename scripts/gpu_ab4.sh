#!/bin/bash
# same-box A/B: A = OWQ_LIB built from another revision (tools/ab_build.sh), B = the in-tree build
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12" "12288 12288 3 0 15 8 20" "12288 12288 4 128 15 1 20"; do
  for r in 1 2; do
    echo -n "A "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape | cut -c1-60
    echo -n "B "; timeout 120 python tools/prof_gemv.py $shape | cut -c1-60
  done
done
