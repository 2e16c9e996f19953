#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
export OWQ_LIB=paper_2306_02272_b200/_ab/exp.so
(for sl in 148 296; do
  echo "== slots $sl"
  OWQ_SB_SLOTS=$sl timeout 120 python tools/sb_trace.py 12288 12288 3 0 15 8 | sed -n '/single/,$p'
  OWQ_SB_SLOTS=$sl timeout 120 python tools/sb_trace.py 4096 4096 4 128 4 8 | sed -n '/single/,$p'
  for a in "11008 4096 4 128 1 8" "4096 4096 4 128 4 8" "4096 11008 4 128 4 8" "12288 12288 3 0 15 16"; do OWQ_SB_SLOTS=$sl timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16" ; done
done) 2>&1 | grep -v "owq sb" | tee gpurun_out/sb13.txt
