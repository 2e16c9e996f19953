#!/bin/bash
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 200 2>&1 | tail -1
(for rep in 1 2; do for B in 1 4 8 16; do
  for L in old sl; do echo -n "$L rep$rep "; OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24; done
  echo -n "cur rep$rep "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done; done) 2>&1 | tee gpurun_out/abold4.txt
