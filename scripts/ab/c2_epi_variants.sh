#!/bin/bash
# C2 K = 1792 scattered-output GEMMs: direct vs staged epilogue vs wide tiles
for m in l2 dx; do for v in direct staged wide; do
  unset SMOE_TC_STAGE_K SMOE_TC_WIDE_MIN_K
  [ $v = staged ] && export SMOE_TC_STAGE_K=2048
  [ $v = wide ] && export SMOE_TC_WIDE_MIN_K=1024
  SMOE_PROF_CFG=C2 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_write.sum --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/c2v_${m}_$v.csv python scripts/prof_one.py $m > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/c2v_${m}_$v.csv | tail -1 | sed "s/^/C2 $m $v /"
done; done
