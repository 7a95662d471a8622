#!/bin/bash
# Tensor-pipe activity with and without epilogue work (SMOE_TC_TIMING=6 = epilogue skipped)
for cfg in C2 C1; do for m in l2 dx rows; do for t in 0 6; do
  SMOE_PROF_CFG=$cfg SMOE_TC_TIMING=$t timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/ep_${cfg}_${m}_$t.csv python scripts/prof_one.py $m > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/ep_${cfg}_${m}_$t.csv | tail -1 | sed "s/^/$cfg $m timing=$t /"
done; done; done
