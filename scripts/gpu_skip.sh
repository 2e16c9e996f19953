#!/bin/bash
for sk in 0 1 2; do
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 40
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 12
  echo -n "SKIP=$sk "; OWQ_SKIP=$sk timeout 120 python tools/prof_gemv.py 4096 4096 3 0 5 1 40
done
