#!/bin/bash
# ncu DRAM bytes + time of the two weight-gradient GEMMs for several raster bands.
for g in 1 2 4 8 16 32; do
  SMOE_GROUP_M_K=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control base -k regex:gemm --csv --log-file gpurun_out/xty_g$g.csv python scripts/prof_one.py xtyboth > /dev/null 2>&1
done
