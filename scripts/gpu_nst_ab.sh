#!/bin/bash
# product-vs-product A/B of the ring-stage cap (8 = product; 6, 12 = _ab builds with only that constant changed)
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
(for s in "12288 12288 3 0 15 1 24" "49152 12288 3 0 3 1 8" "12288 49152 3 0 15 1 8" "12288 12288 3 0 15 8 24"; do
  echo -n "nst8  "; timeout 120 python tools/prof_gemv.py $s
  for n in 6 12; do echo -n "nst$n "; OWQ_LIB=paper_2306_02272_b200/_ab/nst$n.so timeout 120 python tools/prof_gemv.py $s; done
done) 2>&1 | tee gpurun_out/nst_ab.txt
for i in 1 2; do for n in 8 6 12; do
  if [ $n = 8 ]; then timeout 300 python bench.py > gpurun_out/bn_${n}_${i}.json 2>/dev/null; f=gpurun_out/bn_${n}_${i}.json
  else OWQ_LIB=paper_2306_02272_b200/_ab/nst$n.so timeout 300 python bench.py > gpurun_out/bn${n}_${i}.json 2>/dev/null; f=gpurun_out/bn${n}_${i}.json; fi
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('bench nst$n', $i, d['value'], d['ms_per_step'])"
done; done 2>&1 | tee -a gpurun_out/nst_ab.txt
