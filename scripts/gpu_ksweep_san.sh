#!/bin/bash
# weak-column overhead sweep (k in {0, 15, 76, 153} = 3, 3.01, 3.05, 3.1 bits) and compute-sanitizer
mkdir -p gpurun_out
for L in 3 4; do for s in "12288 12288" "49152 12288"; do for k in 0 15 76 153; do
  timeout 120 python tools/prof_gemv.py $s 3 0 $k 1 24 $L; done; done; done 2>&1 | tee gpurun_out/ksweep.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
