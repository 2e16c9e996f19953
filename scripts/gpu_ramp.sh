#!/bin/bash
# ring-fill experiment: OWQ_RAMP = stages in flight while the ring fills (0 = all at once)
for shape in "12288 12288 3 0 15 1 40" "49152 12288 3 0 3 1 12" "12288 12288 3 0 15 8 20" "12288 12288 4 128 15 1 20"; do
  for r in 0 1 2 3 0; do
    echo -n "ramp$r "; OWQ_RAMP=$r timeout 120 python tools/prof_gemv.py $shape | cut -c1-60
  done
done
OWQ_RAMP=2 timeout 120 python tools/trace_graph.py 12288 12288 3 0 15 1 6 2>&1 | head -16
