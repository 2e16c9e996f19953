#!/bin/bash
# round-2 final: GPU suite, smoke, bench (default flags), launch list, ncu of the batched kernel
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/final_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref rc=$?"
for a in "11008 4096 4 128 1 8" "11008 4096 4 128 1 32" "12288 12288 4 128 15 8"; do timeout 120 python tools/prof_batch.py $a 24; done 2>&1 | tee gpurun_out/final_sb.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:owq_gemm_sb -c 1 -f --launch-skip 10 -o gpurun_out/prof_r2_sb_llama_up_b8_v2 python tools/prof_batch.py 11008 4096 4 128 1 8 12 > /dev/null 2>&1; echo "ncu sb rc=$?"
