#!/bin/bash
# DRAM bytes of the wide C1 layer-2 GEMM (K = 14336) per raster band height
# (SMOE_GROUP_M in 128-row units: 8 -> 2 wide blocks ... 64 -> 16), and the
# energy per launch at three of them.
for g in 4 8 16 32 64; do
  SMOE_GROUP_M=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm -c 2 --csv --log-file gpurun_out/bw_g$g.csv python scripts/prof_one.py l2 > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/bw_g$g.csv | tail -1 | sed "s/^/g=$g /"
done
for g in 8 16 32; do SMOE_GROUP_M=$g timeout 100 python scripts/energy.py l2 | sed "s/^/g=$g /"; done
