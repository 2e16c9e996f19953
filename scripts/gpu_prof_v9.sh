#!/bin/bash
timeout 300 ncu --set full --import-source on -k regex:owq_gemv_kernel --launch-skip 20 -c 1 -o gpurun_out/prof_v9c -f python tools/prof_gemv.py 12288 12288 3 0 15 1 20 > gpurun_out/ncu_v9c.log 2>&1; tail -2 gpurun_out/ncu_v9c.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_gemv.py 12288 12288 3 0 15 1 20 > gpurun_out/launches_v9c.csv 2>&1; grep -c owq gpurun_out/launches_v9c.csv
