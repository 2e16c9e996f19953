#!/bin/bash
export OWQ_LIB=paper_2306_02272_b200/_ab/libowq_exp.so
for f in 1 0; do echo "=== fdig=$f"; OWQ_FDIG=$f timeout 120 python tools/trace_graph.py 49152 12288 3 0 3 1 4 2>&1 | head -26; done
