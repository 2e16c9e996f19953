#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
./tools/occ_probe 2>&1 | tee gpurun_out/occ_probe.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/full2_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/full2_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full2_bench.json 2> gpurun_out/full2_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/full2_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None)"
