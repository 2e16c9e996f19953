#!/bin/bash
# relaxed exchanges (product) vs deferred check vs the unbounded lowest summer vs the highest summer
mkdir -p gpurun_out
python -m paper_2306_02272_b200.build > /dev/null
echo "== product parity"; timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 200 2>&1 | tail -1
for L in expnew expdefer; do echo "== $L hand-on forced"; OWQ_SPIN_NS=0 OWQ_LIB=paper_2306_02272_b200/_ab/$L.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_gaps.py -x -q --timeout 200 2>&1 | tail -1; done
(for rep in 1 2; do for B in 1 4 8 16; do
  echo -n "new     "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "defer   "; OWQ_LIB=paper_2306_02272_b200/_ab/expdefer.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "low-unb "; OWQ_LIB=paper_2306_02272_b200/_ab/expsl.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
  echo -n "high    "; OWQ_LIB=paper_2306_02272_b200/_ab/exp.so timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 $B 24
done; done) 2>&1 | tee gpurun_out/handon2.txt
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_handon2_$i.json 2> gpurun_out/bench_handon2_$i.err; head -c 330 gpurun_out/bench_handon2_$i.json | tail -c 130; echo; done
