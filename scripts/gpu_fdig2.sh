#!/bin/bash
export OWQ_LIB=paper_2306_02272_b200/_ab/libowq_exp.so
for e in 0 5 6; do for s in "49152 12288 3 0 3 1 12" "12288 12288 3 0 15 1 40"; do echo -n "exp=$e "; OWQ_EXP=$e timeout 120 python tools/prof_gemv.py $s; done; done
echo -n "fdig0 "; OWQ_FDIG=0 timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 12
