#!/bin/bash
# ncu DRAM bytes + time of the two C1 weight-gradient GEMMs (prof_one.py xtyboth:
# dW2-shaped hT.xg then dW1-shaped xgT.h, 3 reps each) for several raster bands.
# Usage: scripts/ab/xty_sweep.sh [g ...]
gs=${*:-1 2 4 8 16}
for g in $gs; do
  SMOE_GROUP_M_K=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm --csv --log-file gpurun_out/xty_g$g.csv python scripts/prof_one.py xtyboth > /dev/null 2>&1
done
