#!/bin/bash
echo -n "base "; timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
echo -n "N16 "; OWQ_MINN=16 timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
echo -n "noSTTM "; OWQ_EXP=3 timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
echo "== trace N16"; OWQ_MINN=16 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -9
echo "== trace noSTTM"; OWQ_EXP=3 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -9
