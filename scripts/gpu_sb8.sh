#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
timeout 600 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
(for sk in 0 63; do
  echo "== skip $sk"; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so OWQ_SB_SKIP=$sk timeout 120 python tools/sb_trace.py 12288 12288 3 0 15 8 | sed -n '2,12p;60,64p;/graph:/p'
done
for a in "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16"; do timeout 120 python tools/prof_batch.py $a 24 | grep f16; done) 2>&1 | tee gpurun_out/sb8.txt
