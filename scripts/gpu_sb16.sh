#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp_base.so > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_SB_MINB=3 -D OWQ_SB_NST=3 --out paper_2306_02272_b200/_ab/exp_3.so > /dev/null
(for L in exp_base exp_3; do
  echo "== $L"
  for a in "11008 4096 4 128 1 4" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16" "4096 4096 4 128 4 8" "4096 11008 4 128 4 8" "12288 12288 4 128 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 32"; do OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16\|owq sb" | sort -u ; done
done) 2>&1 | tee gpurun_out/sb16.txt
OWQ_LIB=paper_2306_02272_b200/_ab/exp_3.so timeout 300 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
