#!/bin/bash
mkdir -p gpurun_out
for v in "" X0N16 X0N12 NW12; do
  lib=paper_2306_02272_b200/libowq.so; [ -n "$v" ] && lib=paper_2306_02272_b200/_ab/libowq_$v.so
  for shape in "49152 12288 3 0 3 1 12 4" "12288 12288 3 0 15 1 40 4"; do echo -n "[$v] "; OWQ_LIB=$lib timeout 120 python tools/prof_gemv.py $shape; done
done 2>&1 | tee gpurun_out/cc_ab4.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:owq_gemv_cc --launch-skip 6 -c 1 -o gpurun_out/prof_cc2_fc1 -f python tools/prof_gemv.py 49152 12288 3 0 3 1 4 4 > gpurun_out/ncu_cc2_fc1.log 2>&1; echo "ncu rc=$?"
