#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -p no:cacheprovider > gpurun_out/var1.txt 2>&1; echo "variants rc=$?"; tail -25 gpurun_out/var1.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cc" > gpurun_out/var1b.txt 2>&1; echo "cc parity rc=$?"; tail -3 gpurun_out/var1b.txt
