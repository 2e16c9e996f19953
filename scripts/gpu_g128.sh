#!/bin/bash
# grouped-scale (g128) layers at batch 1..16 (BASELINE config 3 shapes and 12288^2), A/B against OWQ_LIB=A
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for shape in "4096 4096 4 128 4 4 40" "4096 4096 4 128 4 16 40" "11008 4096 4 128 1 8 40" "12288 12288 4 128 15 4 20" "12288 12288 4 128 15 1 20" "12288 12288 3 0 15 4 20"; do
  echo -n "A "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape | cut -c1-66
  echo -n "B "; timeout 120 python tools/prof_gemv.py $shape | cut -c1-66
done
