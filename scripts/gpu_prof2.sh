#!/bin/bash
mkdir -p gpurun_out
OWQ_CFG=0 timeout 60 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 2>&1 | tail -2
OWQ_CFG=1 timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > gpurun_out/prof_plain.txt 2>&1 && \
OWQ_CFG=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel -s 3 -c 1 -o gpurun_out/prof_gemv2 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
