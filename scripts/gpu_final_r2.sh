#!/bin/bash
# round-2 close: product library, full GPU suite, smoke, default bench (x2), launch list
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
echo "== -m gpu"; timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_final_$i.json 2> gpurun_out/bench_final_$i.err; done
python - <<'PY'
import json
for i in (1, 2):
    d = json.loads(open(f"gpurun_out/bench_final_{i}.json").read().strip().splitlines()[-1])
    print(i, d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"], d["e2e"]["value"], d.get("gpu_launches"))
PY
