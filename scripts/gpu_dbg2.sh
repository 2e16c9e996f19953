#!/bin/bash
for d in 0 1 2 3; do echo -n "DEBUG=$d "; OWQ_DEBUG=$d timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20; done
echo -n "DEBUG=1+NST8 "; OWQ_NST=8 OWQ_DEBUG=1 timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20
OWQ_DEBUG=1 timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | grep -E "wait|/"
