#!/bin/bash
for d in 0 4 5; do echo -n "DEBUG=$d "; OWQ_DEBUG=$d timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20; done
for d in 4 5; do echo "== trace DEBUG=$d"; OWQ_DEBUG=$d timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 | head -12; done
