#!/bin/bash
# round-2 final (after the prefill row-block selection): suite, smoke, bench, prefill ncu
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final2_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/final2_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench_final.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"
for a in "12288 12288 2048" "49152 12288 1024" "4096 4096 2048" "12288 12288 256" "4096 4096 256" "11008 4096 128"; do timeout 120 python tools/prof_prefill.py $a 4; done 2>&1 | tee gpurun_out/final2_pf.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:owq_prefill -c 1 -f -o gpurun_out/prof_r2_prefill_v3 python tools/prof_prefill.py 12288 12288 2048 1 > /dev/null 2>&1; echo "ncu rc=$?"
