#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-secondary --no-cpu > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo "torchrun rc=$?"; tail -c 400 gpurun_out/torchrun1.json
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "default bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2_bench_default.json')); print(d['value'], d['ms_per_step'], d['steps'], d['warmup'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
