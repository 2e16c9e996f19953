#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:owq_prefill -c 1 -f -o gpurun_out/prof_r2_prefill_v2 python tools/prof_prefill.py 12288 12288 2048 1 > gpurun_out/pf6_ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/prof_r2_prefill_v2.ncu-rep
