#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$? wall=$SECONDS"; tail -2 gpurun_out/r2_bench.err
tail -c 4000 gpurun_out/r2_bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 400 gpurun_out/r2_bench_ref.json
