#!/bin/bash
A=$PWD/paper_2306_02272_b200/_ab/libowq_a.so
shape="49152 12288 3 0 3 1 12"
echo -n "A       "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape
for n in 2 3 4 5 6; do echo -n "B nst=$n "; OWQ_NST=$n timeout 120 python tools/prof_gemv.py $shape; done
for n in 3 4; do echo -n "A nst=$n "; OWQ_LIB=$A OWQ_NST=$n timeout 120 python tools/prof_gemv.py $shape; done
shape="12288 12288 3 0 15 1 40"
echo -n "A       "; OWQ_LIB=$A timeout 120 python tools/prof_gemv.py $shape
for n in 3 4 5; do echo -n "B nst=$n "; OWQ_NST=$n timeout 120 python tools/prof_gemv.py $shape; done
