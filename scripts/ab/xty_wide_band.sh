#!/bin/bash
# Wide dW GEMMs (C1): raster band (SMOE_GROUP_M_K in 256-row blocks; wide tiles use half) vs DRAM bytes and energy
for g in 2 4 8 16 32; do
  SMOE_GROUP_M_K=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm --csv --log-file gpurun_out/xwb_$g.csv python scripts/prof_one.py xtyboth > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/xwb_$g.csv | tail -2 | sed "s/^/g=$g /"
done
for g in 4 8 16; do SMOE_GROUP_M_K=$g timeout 100 python scripts/energy.py xty | sed "s/^/g=$g /"; done
