#!/bin/bash
timeout 300 ncu --set full --import-source on -k regex:owq_gemv_kernel --launch-skip 20 -c 1 -o gpurun_out/prof_v13 -f python tools/prof_gemv.py 12288 12288 3 0 15 1 20 > gpurun_out/ncu_v13.log 2>&1; tail -1 gpurun_out/ncu_v13.log
