timeout 120 python tools/trace_gemv.py 49152 12288 3 0 3 1 2>&1 | head -24
timeout 120 python tools/trace_graph.py 49152 12288 3 0 3 1 4 2>&1 | tail -14
