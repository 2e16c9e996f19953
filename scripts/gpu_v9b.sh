#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 8 20
timeout 300 ncu --set full --import-source on -k regex:owq_gemv_kernel --launch-skip 20 -c 1 -o gpurun_out/prof_v9 -f python tools/prof_gemv.py 12288 12288 3 0 15 1 20 > gpurun_out/ncu_v9.log 2>&1; tail -3 gpurun_out/ncu_v9.log
