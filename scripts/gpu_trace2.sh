timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | tail -15
timeout 120 python tools/trace_graph.py 12288 12288 3 0 15 1 6 2>&1 | tail -15
