#!/bin/bash
export OWQ_LIB=paper_2306_02272_b200/_ab/libowq_exp.so
for pdl in 2 1 0; do for s in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12"; do echo -n "pdl=$pdl "; OWQ_PDL=$pdl timeout 120 python tools/prof_gemv.py $s; done; done
for nst in 3 4 6; do for s in "12288 12288 3 0 15 1 40"; do echo -n "nst=$nst "; OWQ_NST=$nst timeout 120 python tools/prof_gemv.py $s; done; done
