#!/bin/bash
mkdir -p gpurun_out
for mb in 1 2; do
  echo "MINB=$mb"
  for shp in "12288 12288 3 0 15 1 20" "49152 12288 3 0 3 1 10" "12288 49152 3 0 15 1 10" "4096 4096 4 128 4 1 50"; do
    OWQ_MINB=$mb timeout 120 python tools/prof_gemv.py $shp
  done
done > gpurun_out/exp.txt 2>&1
OWQ_MINB=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "parity or stream_k or probes" --timeout 300 > gpurun_out/exp_pytest.log 2>&1
OWQ_MINB=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "parity or stream_k or probes" --timeout 300 >> gpurun_out/exp_pytest.log 2>&1
cat gpurun_out/exp.txt; grep -E "passed|failed" gpurun_out/exp_pytest.log
