#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pf9_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pf9_tests.txt
