#!/bin/bash
for d in 0 6; do echo -n "DEBUG=$d "; OWQ_DEBUG=$d timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20; done
for d in 6; do echo "== trace DEBUG=$d"; OWQ_DEBUG=$d timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -14; done
