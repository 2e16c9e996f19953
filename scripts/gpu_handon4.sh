#!/bin/bash
# protocol by batch (highest summer B <= 3, bounded lowest B >= 4): GPU suite, forced
# hand-on at every B, bench A/B against the highest-summer-only library (3517d2a)
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
echo "== product -m gpu"; timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -1
echo "== hand-on forced at every B (OWQ_LOW_MINB=1 OWQ_SPIN_NS=0)"; OWQ_LOW_MINB=1 OWQ_SPIN_NS=0 OWQ_LIB=paper_2306_02272_b200/_ab/expnew.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 200 2>&1 | tail -1
for i in 1 2 3; do
  timeout 300 python bench.py > gpurun_out/bench4_new_$i.json 2> gpurun_out/bench4_new_$i.err
  OWQ_LIB=paper_2306_02272_b200/_ab/high.so timeout 300 python bench.py > gpurun_out/bench4_high_$i.json 2> gpurun_out/bench4_high_$i.err
done
python - <<'PY'
import json
for k in ("new", "high"):
    for i in (1, 2, 3):
        d = json.loads(open(f"gpurun_out/bench4_{k}_{i}.json").read().strip().splitlines()[-1])
        print(k, i, d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
(for B in 1 4 8 16; do
  echo -n "new  "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "high "; OWQ_LIB=paper_2306_02272_b200/_ab/high.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done) 2>&1 | tee gpurun_out/handon4.txt
