#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel -s 3 -c 1 -o gpurun_out/prof_v6 python tools/prof_gemv.py 12288 12288 3 0 15 1 4 > gpurun_out/ncu_v6.log 2>&1
tail -1 gpurun_out/ncu_v6.log
