#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 10
timeout 120 python tools/prof_gemv.py 12288 12288 4 0 15 1 20
echo "== trace"; timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -12
timeout 300 ncu --set full --import-source on -k regex:owq_gemv_kernel --launch-skip 20 -c 1 -o gpurun_out/prof_v12 -f python tools/prof_gemv.py 12288 12288 3 0 15 1 20 > gpurun_out/ncu_v12.log 2>&1; tail -1 gpurun_out/ncu_v12.log
