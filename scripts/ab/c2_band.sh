#!/bin/bash
# C2 layer-2 GEMM (K = 1792): raster band height vs time / DRAM / MMA lfull wait
for g in 2 4 8 16 32 64; do
  SMOE_PROF_CFG=C2 SMOE_GROUP_M=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/c2b_$g.csv python scripts/prof_one.py l2 > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/c2b_$g.csv | tail -1 | sed "s/^/g=$g /"
  SMOE_PROF_CFG=C2 SMOE_GROUP_M=$g SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py l2 2>&1 | grep "timing cluster" | tail -1 | sed "s/^/g=$g /"
done
