#!/bin/bash
mkdir -p gpurun_out
OWQ_DWG=${DWG:-2} timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | tee gpurun_out/trace2.txt
