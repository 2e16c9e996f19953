#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ldig1_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ldig1_tests.txt
(for L in 0 1; do
  echo "== OWQ_LDIG=$L"
  for a in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12" "4096 4096 3 0 5 1 40" "9216 9216 3 0 11 1 40"; do OWQ_LDIG=$L OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $a; done
done) 2>&1 | tee gpurun_out/ldig1_time.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu > gpurun_out/ldig1_bench.json 2> gpurun_out/ldig1_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/ldig1_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], {k: v['us'] for k, v in d['us_per_layer'].items()})"
