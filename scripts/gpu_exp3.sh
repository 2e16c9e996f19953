#!/bin/bash
mkdir -p gpurun_out
for cfg in 0 1; do for dbg in 0 1; do
  echo "== CFG=$cfg DEBUG=$dbg"; OWQ_CFG=$cfg OWQ_DEBUG=$dbg timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
  OWQ_CFG=$cfg OWQ_DEBUG=$dbg timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1
done; done 2>&1 | tee gpurun_out/exp3.txt
