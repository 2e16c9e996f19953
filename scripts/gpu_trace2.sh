timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | tail -12
