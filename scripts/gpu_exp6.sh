#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for dwg in 3 2; do
  for shp in "12288 12288 3 0 15 1 20" "49152 12288 3 0 3 1 10" "12288 49152 3 0 15 1 10" "4096 4096 4 128 4 1 50"; do
    echo -n "DWG=$dwg "; OWQ_DWG=$dwg timeout 120 python tools/prof_gemv.py $shp
  done
done 2>&1 | tee gpurun_out/exp6.txt
OWQ_DWG=3 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | grep -E "CTAs|start|fin|end|wait|/"
