#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
for r in 1 2; do
  for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "4096 4096 3 0 5 1 40" "12288 12288 3 0 15 2 40" "12288 12288 3 0 15 4 40"; do
    echo -n "A "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape
    echo -n "B "; timeout 120 python tools/prof_gemv.py $shape
  done
done
echo "== trace B fc1"; OWQ_SKIP=1 timeout 120 python tools/trace_gemv.py 49152 12288 3 0 3 1 2>&1 | sed -n "1,3p;19,22p"
