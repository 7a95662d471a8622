#!/bin/bash
# C3 projection GEMMs: MMA-issuer wait counters and tensor-pipe activity
for m in gathers ofwd; do
  echo "== C3 $m"; SMOE_PROF_CFG=C3 SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py $m 2>&1 | grep "timing cluster" | tail -2
  SMOE_PROF_CFG=C3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/c3_$m.csv python scripts/prof_one.py $m > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/c3_$m.csv | tail -1
  SMOE_PROF_CFG=C3 SMOE_TC_TIMING=6 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/c3_${m}_noepi.csv python scripts/prof_one.py $m > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/c3_${m}_noepi.csv | tail -1 | sed 's/^/no-epilogue: /'
done
