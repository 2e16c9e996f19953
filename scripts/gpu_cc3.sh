#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -q -x -p no:cacheprovider -k "cc" > gpurun_out/cc_par3.txt 2>&1; echo "cc parity rc=$?"; tail -4 gpurun_out/cc_par3.txt
for v in "" NW12 MINB2 NW16 S2 S8; do
  lib=paper_2306_02272_b200/libowq.so; [ -n "$v" ] && lib=paper_2306_02272_b200/_ab/libowq_$v.so
  for shape in "49152 12288 3 0 3 1 12 4" "12288 12288 3 0 15 1 40 4" "12288 12288 4 128 15 1 40 4"; do echo -n "[$v] "; OWQ_LIB=$lib timeout 120 python tools/prof_gemv.py $shape; done
done 2>&1 | tee gpurun_out/cc_ab3.txt
