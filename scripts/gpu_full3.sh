#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/full3_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/full3_tests.txt
for a in "12288 12288 2048" "49152 12288 1024" "4096 4096 2048" "12288 12288 256"; do timeout 120 python tools/prof_prefill.py $a 4; done 2>&1 | tee gpurun_out/full3_pf.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
