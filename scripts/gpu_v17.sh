#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 10
timeout 120 python tools/prof_gemv.py 12288 49152 3 0 15 1 10
timeout 120 python tools/prof_gemv.py 12288 12288 4 0 15 1 20
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 2 20
timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 8 20
echo "== trace"; timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | sed -n '1,8p;20,30p'
