#!/bin/bash
mkdir -p gpurun_out
for dbg in 0 1; do echo "== DEBUG=$dbg"; OWQ_DEBUG=$dbg timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1; done 2>&1 | tee gpurun_out/trace.txt
