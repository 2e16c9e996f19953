#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/final4_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/final4_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:owq_prefill_kernel -c 1 -f -o gpurun_out/prof_r2_prefill_v4 python tools/prof_prefill.py 12288 12288 2048 1 1 > /dev/null 2>&1; echo "ncu rc=$?"
