#!/bin/bash
# round-2 profiles: launch list of the bench (cold, serialised) + one --set full capture per kernel / shape
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
NCU="ncu --set full --clock-control none --import-source on -c 1 -f"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv \
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 30 -o gpurun_out/prof_r2_q python tools/prof_gemv.py 12288 12288 3 0 15 1 40 > /dev/null 2>&1; echo "q rc=$?"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 10 -o gpurun_out/prof_r2_fc1 python tools/prof_gemv.py 49152 12288 3 0 3 1 12 > /dev/null 2>&1; echo "fc1 rc=$?"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 10 -o gpurun_out/prof_r2_fc2 python tools/prof_gemv.py 12288 49152 3 0 15 1 12 > /dev/null 2>&1; echo "fc2 rc=$?"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 20 -o gpurun_out/prof_r2_b8 python tools/prof_gemv.py 12288 12288 3 0 15 8 20 > /dev/null 2>&1; echo "b8 rc=$?"
ls -la gpurun_out/*.ncu-rep
