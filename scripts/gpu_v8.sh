#!/bin/bash
# v8 kernel: parity, then timing variants (DWG, items per WG per stage)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for dwg in 3 4; do for ipw in 2 3 4; do
  echo -n "DWG=$dwg IPW=$ipw "; OWQ_DWG=$dwg OWQ_IPW=$ipw timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
done; done
for dwg in 3 4; do
  echo -n "DWG=$dwg "; OWQ_DWG=$dwg timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 10
  echo -n "DWG=$dwg "; OWQ_DWG=$dwg timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 8 20
  echo -n "DWG=$dwg "; OWQ_DWG=$dwg timeout 120 python tools/prof_gemv.py 12288 12288 4 128 15 1 20
done
echo "== trace DWG=3"; OWQ_DWG=3 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -24
