#!/bin/bash
mkdir -p gpurun_out
export OWQ_LIB=paper_2306_02272_b200/_ab/libowq_exp.so
timeout 120 python tools/trace_graph.py 12288 12288 3 0 15 1 6 > gpurun_out/trace_q.txt 2>&1; echo rc=$?; cat gpurun_out/trace_q.txt
timeout 120 python tools/trace_graph.py 49152 12288 3 0 3 1 4 > gpurun_out/trace_fc1.txt 2>&1; echo rc=$?; head -30 gpurun_out/trace_fc1.txt
for skip in 0 1; do for s in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12"; do echo -n "skip=$skip "; OWQ_SKIP=$skip timeout 120 python tools/prof_gemv.py $s; done; done
