#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
OWQ_FORCE_COUNTER=1 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 200 2>&1 | tail -1
(for B in 1 2 4 8 16; do
  echo -n "exp-slot-new "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "exp-slot-low "; OWQ_LIB=paper_2306_02272_b200/_ab/expsl.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "exp-counter  "; OWQ_FORCE_COUNTER=1 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done
for L in exp expsl; do echo -n "$L fc1 "; OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 8; done
echo -n "counter fc1 "; OWQ_FORCE_COUNTER=1 OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 8) 2>&1 | tee gpurun_out/counter.txt
