#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for cfg in 0 1; do
  for shp in "12288 12288 3 0 15 1 20" "49152 12288 3 0 3 1 10" "4096 4096 4 128 4 1 50"; do
    echo -n "CFG=$cfg "; OWQ_CFG=$cfg timeout 120 python tools/prof_gemv.py $shp
  done
  echo -n "CFG=$cfg DEBUG=1 "; OWQ_DEBUG=1 OWQ_CFG=$cfg timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
done 2>&1 | tee gpurun_out/exp2.txt
OWQ_CFG=0 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | tee gpurun_out/trace.txt
