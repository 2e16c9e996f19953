#!/bin/bash
for m in 0 1 2; do
  echo -n "PDL=$m "; OWQ_PDL=$m timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 40
  echo -n "PDL=$m "; OWQ_PDL=$m timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 12
done
