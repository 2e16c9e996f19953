#!/bin/bash
# bounded-wait lowest-piece fixup: parity (product; experiment build with the
# hand-on path forced by OWQ_SPIN_NS=0), A/B against the previous protocols, bench
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
echo "== product parity"; timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
echo "== hand-on forced (OWQ_SPIN_NS=0)"; OWQ_SPIN_NS=0 OWQ_LIB=paper_2306_02272_b200/_ab/expnew.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 200 2>&1 | tail -1
(for B in 1 2 4 8 16; do
  echo -n "new       "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "high      "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "low-unb   "; OWQ_LIB=paper_2306_02272_b200/_ab/expsl.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "new-spin0 "; OWQ_SPIN_NS=0 OWQ_LIB=paper_2306_02272_b200/_ab/expnew.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done
for s in "49152 12288 3 0 3 1 8" "12288 49152 3 0 15 1 8" "4096 4096 4 128 4 1 40" "11008 4096 4 128 1 8 40"; do
  echo -n "new  "; timeout 120 python tools/prof_gemv.py $s
  echo -n "high "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py $s
done) 2>&1 | tee gpurun_out/handon.txt
timeout 300 python bench.py > gpurun_out/bench_handon.json 2> gpurun_out/bench_handon.err; tail -c 600 gpurun_out/bench_handon.json
