#!/bin/bash
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for shape in "49152 12288 3 0 3 1 12" "12288 12288 3 0 15 1 40"; do
for d in 2 3 4; do
  echo -n "A dwg=$d "; OWQ_LIB=$A OWQ_DWG=$d timeout 120 python tools/prof_gemv.py $shape
  echo -n "B dwg=$d "; OWQ_DWG=$d timeout 120 python tools/prof_gemv.py $shape
done; done
