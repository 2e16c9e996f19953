#!/bin/bash
# final: full GPU suite on the bounded-wait lowest-piece fixup; bench A/B on one box
# against the previous product protocol (highest-index summer, commit 3517d2a); launch list
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
echo "== product -m gpu"; timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -1
for i in 1 2 3; do
  timeout 300 python bench.py > gpurun_out/bench_new_$i.json 2> gpurun_out/bench_new_$i.err
  OWQ_LIB=paper_2306_02272_b200/_ab/high.so timeout 300 python bench.py > gpurun_out/bench_high_$i.json 2> gpurun_out/bench_high_$i.err
done
python - <<'PY'
import json
for k in ("new", "high"):
    for i in (1, 2, 3):
        d = json.loads(open(f"gpurun_out/bench_{k}_{i}.json").read().strip().splitlines()[-1])
        print(k, i, d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches_final.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_final.log 2>&1; echo "ncu rc $?"
