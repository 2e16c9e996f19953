#!/bin/bash
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.sh
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
echo "== A"; OWQ_LIB=$A timeout 120 python tools/trace_gemv.py 49152 12288 3 0 3 1 2>&1 | sed -n '1,5p;19,22p'
echo "== B"; timeout 120 python tools/trace_gemv.py 49152 12288 3 0 3 1 2>&1 | sed -n '1,5p;19,22p'
