#!/bin/bash
python -m paper_2306_02272_b200.build > /dev/null
# both layouts: fixed-cost sweep (M x 12288, 3-bit per-row) and BASELINE config shapes
mkdir -p gpurun_out
for L in 3 4; do
  for M in 3072 6144 12288 24576 49152; do timeout 120 python tools/prof_gemv.py $M 12288 3 0 15 1 24 $L; done
  for s in "12288 49152 3 0 15 1 12" "4096 4096 3 0 5 1 40" "16384 4096 3 0 1 1 40" "4096 16384 3 0 5 1 40" \
           "9216 9216 3 0 11 1 40" "36864 9216 3 0 2 1 16" "9216 36864 3 0 11 1 16" \
           "12288 12288 4 128 15 1 24" "4096 4096 4 128 4 1 40" "11008 4096 4 128 1 1 40" "4096 11008 4 128 4 1 40" \
           "12288 12288 3 0 15 2 24" "12288 12288 3 0 15 4 24" "12288 12288 3 0 15 8 24" "12288 12288 3 0 15 16 24" \
           "11008 4096 4 128 1 4 40" "11008 4096 4 128 1 8 40" "11008 4096 4 128 1 16 40"; do
    timeout 120 python tools/prof_gemv.py $s $L
  done
done 2>&1 | tee gpurun_out/table3.txt
