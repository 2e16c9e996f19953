#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
python -m paper_2306_02272_b200.build -D OWQ_EXPERIMENTS --out paper_2306_02272_b200/_ab/exp.so > /dev/null
for sk in auto 0 8 15 25; do
  if [ "$sk" = auto ]; then unset OWQ_SKEW; else export OWQ_SKEW=$sk; fi
  OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 600 python bench.py --steps 50 --warmup 10 --no-secondary --no-cpu --no-e2e > gpurun_out/skew5_$sk.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/skew5_$sk.json')); print('skew $sk', d['value'], d['ms_per_step'], {k: v['us'] for k, v in d['us_per_layer'].items()})"
done 2>&1 | tee gpurun_out/skew5.txt
