#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS -D OWQ_SB_SPIN=1 --out paper_2306_02272_b200/_ab/exp_spin.so > /dev/null
(for L in exp exp_spin; do
  echo "== $L"
  for sk in 0 63; do echo "skip $sk"; OWQ_SB_SKIP=$sk OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/sb_trace.py 12288 12288 3 0 15 8 2>&1 | sed -n '2,8p;/graph:/p'; done
  for a in "11008 4096 4 128 1 8" "4096 4096 4 128 4 8" "12288 12288 4 128 15 8" "12288 12288 3 0 15 16"; do OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16" ; done
done) 2>&1 | grep -v "owq sb" | tee gpurun_out/sb14.txt
OWQ_LIB=paper_2306_02272_b200/_ab/exp_spin.so timeout 300 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
