#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_SB_SUB=2 --out paper_2306_02272_b200/_ab/sub2.so > /dev/null
timeout 600 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
(for L in libowq _ab/sub2; do
  echo "== $L"
  for a in "12288 12288 3 0 15 8" "12288 12288 3 0 15 16" "11008 4096 4 128 1 4" "11008 4096 4 128 1 8" "11008 4096 4 128 1 16" "12288 12288 4 128 15 8" "4096 4096 4 128 4 8" "49152 12288 3 0 3 8"; do OWQ_LIB=paper_2306_02272_b200/$L.so timeout 120 python tools/prof_batch.py $a 24 2>&1 | grep "f16" ; done
done) 2>&1 | tee gpurun_out/sb12.txt
OWQ_LIB=paper_2306_02272_b200/_ab/sub2.so timeout 600 python -m pytest tests/test_gpu_batch_f16.py -x -q 2>&1 | tail -2
