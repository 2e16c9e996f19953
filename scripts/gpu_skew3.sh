#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/skew3_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/skew3_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/skew3_bench.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/skew3_bench.json')); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], {k: v['us'] for k, v in d['us_per_layer'].items()}, d['clocks'])"
