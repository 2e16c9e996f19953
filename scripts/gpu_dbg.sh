#!/bin/bash
mkdir -p gpurun_out
for dbg in 0 1 2; do
  for shp in "12288 12288 3 0 15 1 20" "49152 12288 3 0 3 1 10"; do
    echo -n "DEBUG=$dbg "; OWQ_DEBUG=$dbg timeout 120 python tools/prof_gemv.py $shp
  done
done > gpurun_out/dbg.txt 2>&1
cat gpurun_out/dbg.txt
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
