#!/bin/bash
# final verification of the committed state: GPU suite, smoke, default bench
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/final3_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/final3_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_final3.json 2> gpurun_out/r2_bench_final3.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench_final3.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e'].get('graphed'), d['clocks'], d['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref3.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/r2_bench_ref3.json
