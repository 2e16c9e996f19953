#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for cfg in 0 1; do
  for shp in "12288 12288 3 0 15 1 20" "49152 12288 3 0 3 1 10"; do
    echo -n "CFG=$cfg "; OWQ_CFG=$cfg timeout 120 python tools/prof_gemv.py $shp
  done
done 2>&1 | tee gpurun_out/exp5.txt
for cfg in 0 1; do
OWQ_CFG=$cfg timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > /dev/null 2>&1 && \
OWQ_CFG=$cfg timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel -s 3 -c 1 -o gpurun_out/prof_cfg$cfg python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > gpurun_out/ncu_cfg$cfg.log 2>&1
tail -1 gpurun_out/ncu_cfg$cfg.log
done
