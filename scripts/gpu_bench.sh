#!/bin/bash
# round-end style: tests, smoke, bench (N=1) + reference arm + launch list + ncu --set full of the three GEMV shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3500 gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel --launch-skip 30 -c 1 -o gpurun_out/prof_r1_q -f python tools/prof_gemv.py 12288 12288 3 0 15 1 40 > gpurun_out/ncu_full_q.log 2>&1; echo "ncu q rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel --launch-skip 10 -c 1 -o gpurun_out/prof_r1_fc1 -f python tools/prof_gemv.py 49152 12288 3 0 3 1 12 > gpurun_out/ncu_full_fc1.log 2>&1; echo "ncu fc1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owq_gemv_kernel --launch-skip 10 -c 1 -o gpurun_out/prof_r1_fc2 -f python tools/prof_gemv.py 12288 49152 3 0 15 1 12 > gpurun_out/ncu_full_fc2.log 2>&1; echo "ncu fc2 rc=$?"
