#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py tests/test_gpu_guards.py -q -x -p no:cacheprovider -k "tc or not cc" > gpurun_out/fdig_t.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/fdig_t.txt
for f in 1 0; do for s in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12" "4096 4096 3 0 5 1 40"; do echo -n "fdig=$f "; OWQ_FDIG=$f OWQ_LIB=paper_2306_02272_b200/_ab/libowq_exp.so timeout 120 python tools/prof_gemv.py $s; done; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-secondary > gpurun_out/fdig_bench.json 2>gpurun_out/fdig_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/fdig_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['step_ms_p10_p50_p90'], {k: v['us'] for k, v in d['us_per_layer'].items()})"
