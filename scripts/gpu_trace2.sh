timeout 120 python tools/trace_gemv.py 12288 12288 4 128 15 1 2>&1 | head -30
