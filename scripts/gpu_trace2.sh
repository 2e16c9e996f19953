#!/bin/bash
# per-CTA timelines: one call (tools/trace_gemv.py) and the last call of a graph of
# back-to-back calls (tools/trace_graph.py), 12288^2 and 49152x12288, batch 1
timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | tail -15
timeout 120 python tools/trace_graph.py 49152 12288 3 0 3 1 4 2>&1 | tail -15
