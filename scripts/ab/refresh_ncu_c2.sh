#!/bin/bash
# ncu --set full of the C2 GEMMs (SMOE_PROF_CFG=C2): DRAM traffic for profiles/traffic.json
mkdir -p gpurun_out
for m in xty l1s dhs l2 dx; do
  SMOE_PROF_CFG=C2 timeout 300 ncu --set full --clock-control none -k regex:tc2_gemm -c 1 -o gpurun_out/rn2_full_$m python scripts/prof_one.py $m > /dev/null 2>&1; echo "full $m rc $?"
  ncu -i gpurun_out/rn2_full_$m.ncu-rep --page raw --csv > gpurun_out/rn2_full_$m.csv 2>/dev/null
  rm -f gpurun_out/rn2_full_$m.ncu-rep
done
