#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/skew2_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/skew2_tests.txt
(for a in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 49152 3 0 15 1 12" "4096 4096 3 0 5 1 40" "9216 9216 3 0 11 1 40" "36864 9216 3 0 2 1 12"; do timeout 120 python tools/prof_gemv.py $a; OWQ_SKEW=0 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $a; done) 2>&1 | tee gpurun_out/skew2.txt
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu > gpurun_out/skew2_bench$i.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/skew2_bench$i.json')); print('bench', d['value'], d['ms_per_step'], {k: v['us'] for k, v in d['us_per_layer'].items()})"; done
for i in 1 2; do OWQ_SKEW=0 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 600 python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu > gpurun_out/skew2_bench0_$i.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/skew2_bench0_$i.json')); print('bench skew0(exp build)', d['value'], d['ms_per_step'])"; done
