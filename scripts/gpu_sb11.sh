#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
for cfg in "1 4" "1 8" "2 4" "2 3" "4 2"; do set -- $cfg
  python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_SB_SUB=$1 -D OWQ_SB_NST=$2 --out paper_2306_02272_b200/_ab/exp_$1_$2.so > /dev/null
done
(for cfg in "1 4" "1 8" "2 4" "2 3" "4 2"; do set -- $cfg
  echo "== SUB=$1 NST=$2"
  for a in "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 8" "12288 12288 4 128 15 8"; do OWQ_LIB=paper_2306_02272_b200/_ab/exp_$1_$2.so timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16\|owq sb" ; done
done) 2>&1 | tee gpurun_out/sb11.txt
