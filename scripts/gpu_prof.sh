#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/mma_probe > gpurun_out/mma_probe.txt 2>&1
timeout 300 python tools/prof_gemv.py > gpurun_out/prof_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel -s 2 -c 1 -o gpurun_out/prof_gemv1 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > gpurun_out/ncu1.log 2>&1
cat gpurun_out/mma_probe.txt gpurun_out/prof_plain.txt; tail -3 gpurun_out/ncu1.log
