#!/bin/bash
# DESIGN.md measurement table: device-timed per-call latency (graph of back-to-back
# calls over rotating weight copies > L2), one line per layer configuration.
python -m paper_2306_02272_b200.build >/dev/null
for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12" \
             "12288 12288 4 0 15 1 40" "12288 12288 4 128 15 1 20" \
             "12288 12288 3 0 15 2 20" "12288 12288 3 0 15 4 20" "12288 12288 3 0 15 8 20" "12288 12288 3 0 15 16 20" \
             "4096 4096 3 0 5 1 40" "4096 4096 4 128 4 1 40" "4096 4096 4 128 4 4 40" "4096 4096 4 128 4 16 40" \
             "11008 4096 4 128 1 8 40"; do
  timeout 120 python tools/prof_gemv.py $shape
done
