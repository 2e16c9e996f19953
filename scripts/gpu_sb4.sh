#!/bin/bash
# batched f16 kernel: which role sets the ~2.4 us per stage (experiment build, OWQ_SB_SKIP)
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
for sk in 0 1 2 4 8 3 5 6 7 15; do
  for a in "11008 4096 4 128 1 8" "12288 12288 3 0 15 8"; do
    echo -n "skip=$sk "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so OWQ_SB_SKIP=$sk timeout 120 python tools/prof_batch.py $a 24 | grep f16
  done
done 2>&1 | tee gpurun_out/sb4_skip.txt
