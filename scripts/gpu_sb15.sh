#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
for cfg in "1 4" "2 2" "1 3" "1 6"; do set -- $cfg
  python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_SB_SUB=$1 -D OWQ_SB_NST=$2 --out paper_2306_02272_b200/_ab/exp_$1_$2.so > /dev/null
done
(for cfg in "1 4" "2 2" "1 3" "1 6"; do set -- $cfg
  echo "== SUB=$1 NST=$2"
  for a in "11008 4096 4 128 1 8" "4096 4096 4 128 4 8" "12288 12288 4 128 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 16"; do OWQ_LIB=paper_2306_02272_b200/_ab/exp_$1_$2.so timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16\|owq sb" | sort -u ; done
done) 2>&1 | tee gpurun_out/sb15.txt
OWQ_LIB=paper_2306_02272_b200/_ab/exp_2_2.so timeout 300 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
