#!/bin/bash
# round-2 profiles: launch list of the bench (cold, serialised) + one --set full capture per kernel / shape
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b_tests.txt
NCU="ncu --set full --clock-control none --import-source on -c 1 -f"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 10 -o gpurun_out/prof_r2_q python tools/prof_gemv.py 12288 12288 3 0 15 1 12 > /dev/null 2>&1; echo "q rc=$?"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 20 -o gpurun_out/prof_r2_b16 python tools/prof_gemv.py 12288 12288 3 0 15 16 20 > /dev/null 2>&1; echo "b16 rc=$?"
timeout 300 $NCU -k regex:owq_gemv_kernel --launch-skip 20 -o gpurun_out/prof_r2_g128 python tools/prof_gemv.py 12288 12288 4 128 15 1 20 > /dev/null 2>&1; echo "g128 rc=$?"
timeout 300 $NCU -k regex:owq_gemv_cc --launch-skip 20 -o gpurun_out/prof_r2_cc_g128 python tools/prof_gemv.py 12288 12288 4 128 15 1 20 4 > /dev/null 2>&1; echo "cc g128 rc=$?"
timeout 300 $NCU -k regex:owq_gemv_cc --launch-skip 20 -o gpurun_out/prof_r2_cc_q python tools/prof_gemv.py 12288 12288 3 0 15 1 20 4 > /dev/null 2>&1; echo "cc q rc=$?"
timeout 300 $NCU -k regex:owq_gemm_sb --launch-skip 10 -o gpurun_out/prof_r2_sb_llama_up_b8 python tools/prof_batch.py 11008 4096 4 128 1 8 12 > /dev/null 2>&1; echo "sb rc=$?"
timeout 300 $NCU -k regex:owq_prefill --launch-skip 3 -o gpurun_out/prof_r2_prefill python tools/prof_prefill.py 12288 12288 2048 4 > /dev/null 2>&1; echo "prefill rc=$?"
ls -la gpurun_out/*.ncu-rep
