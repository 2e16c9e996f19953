#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for sk in 0 1; do
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 40
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 12
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 4096 4096 3 0 5 1 40
done
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 8 20
timeout 120 python tools/prof_gemv.py 12288 12288 4 128 15 1 20
echo "== trace 4096"; OWQ_SKIP=1 timeout 120 python tools/trace_gemv.py 4096 4096 3 0 5 1 2>&1 | sed -n '1,3p;18,40p'
