#!/bin/bash
# MMA-issuer wait counters of the C2 GEMMs (SMOE_TC_TIMING=1)
for m in l1s l2 dx dhs xty; do
  echo "== C2 $m"; SMOE_PROF_CFG=C2 SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py $m 2>&1 | grep "timing cluster" | tail -2
done
for m in l2 dx; do
  SMOE_PROF_CFG=C2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/c2_$m.csv python scripts/prof_one.py $m > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/c2_$m.csv | tail -1 | sed "s/^/C2 $m /"
done
