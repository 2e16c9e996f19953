#!/bin/bash
# Decode sensitivity probe (timing only, results wrong): no digit pass
# (OWQ_SKIP=1); OWQ_EXP 8 = twice the decode math, 16 = twice the TMEM stores.
python -m paper_2306_02272_b200.build >/dev/null
for shape in "49152 12288 3 0 3 1 12"; do
  for e in 0 8 16 24 3; do
    echo -n "exp$e "; OWQ_SKIP=1 OWQ_EXP=$e timeout 120 python tools/prof_gemv.py $shape | cut -c1-60
  done
done
