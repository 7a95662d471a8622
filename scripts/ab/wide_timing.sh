#!/bin/bash
# Issue-loop wait counters (SMOE_TC_TIMING=1) of the C1 GEMMs, 256-row vs wide tiles.
for m in rows l2 dh xty; do for w in 0 1; do
  echo "== $m wide=$w"; SMOE_TC_WIDE=$w SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py $m 2>&1 | grep "timing cluster" | tail -4
done; done
