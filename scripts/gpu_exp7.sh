#!/bin/bash
for e in 0 1 2 3; do echo -n "EXP=$e "; OWQ_EXP=$e timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 20; done
for e in 1 2 3; do echo "== trace EXP=$e"; OWQ_EXP=$e timeout 120 python tools/trace_gemv.py 12288 12288 3 0 15 1 2>&1 | head -10; done
