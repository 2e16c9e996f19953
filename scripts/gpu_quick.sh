#!/bin/bash
# quick GPU iteration: parity subset + per-shape timing + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print("value", d["value"], "GB/s; frac", d["roofline"]["frac"], "clocks", d["clocks"])
for k,v in d["us_per_layer"].items(): print(k, v)
print("e2e", d["e2e"])
PY
tail -2 gpurun_out/bench.err
