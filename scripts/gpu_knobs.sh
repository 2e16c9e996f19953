#!/bin/bash
for ipw in 3 4 5 6; do for nst in 3 4 6; do
  echo -n "ipw=$ipw nst=$nst "; OWQ_IPW=$ipw OWQ_NST=$nst timeout 120 python tools/prof_gemv.py 12288 12288 3 0 15 1 40 | cut -c1-60
  echo -n "ipw=$ipw nst=$nst "; OWQ_IPW=$ipw OWQ_NST=$nst timeout 120 python tools/prof_gemv.py 49152 12288 3 0 3 1 12 | cut -c1-60
done; done
