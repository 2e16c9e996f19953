#!/bin/bash
# round 2, first GPU call: gap parity tests, full gpu suite, box calibration probes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/r2_smi.txt
nproc > gpurun_out/r2_host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/r2_host.txt
timeout 120 ./tools/cc_probe > gpurun_out/r2_cc_probe.txt 2>&1; echo "cc_probe rc=$?"
timeout 120 ./tools/hbm_probe > gpurun_out/r2_hbm_probe.txt 2>&1; echo "hbm_probe rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity_gaps.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r2_gaps.txt 2>&1; echo "gaps rc=$?"; tail -5 gpurun_out/r2_gaps.txt
timeout 900 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_parity_gaps.py -p no:cacheprovider > gpurun_out/r2_gpu.txt 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r2_gpu.txt
for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "4096 4096 3 0 5 1 40"; do timeout 120 python tools/prof_gemv.py $shape; done > gpurun_out/r2_table0.txt 2>&1
cat gpurun_out/r2_cc_probe.txt gpurun_out/r2_hbm_probe.txt gpurun_out/r2_table0.txt
