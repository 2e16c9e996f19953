#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for d in 4 3 2; do
  echo -n "DWG=$d "; OWQ_DWG=$d timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
  echo -n "DWG=$d "; OWQ_DWG=$d timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 10
  echo -n "DWG=$d "; OWQ_DWG=$d timeout 120 python tools/prof_gemv.py 12288 12288 4 0 15 1 20
done
for d in 4 3; do echo "== trace DWG=$d"; OWQ_DWG=$d timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | sed -n '1,8p;20,30p'; done
