#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q --timeout 200 2>&1 | tail -3
(for a in "4096 4096 256" "4096 4096 128" "4096 11008 128" "4096 4096 32" "11008 4096 128" "12288 12288 256" "12288 12288 2048"; do
  timeout 120 python tools/prof_prefill.py $a 4 0; timeout 120 python tools/prof_prefill.py $a 4 1; done) 2>&1 | tee gpurun_out/pf13_time.txt
