#!/bin/bash
# Base-clock ncu of one GEMM mode under several env settings (same session).
# usage: env_sweep.sh TAG MODE "VAR=a VAR2=b" "VAR=c" ...   (each arg = one setting; "-" = none)
tag=$1; m=$2; shift 2
i=0
for setting in "$@"; do
  [ "$setting" = "-" ] && setting=""
  env $setting timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control base -k regex:gemm -s 2 -c 1 --csv --log-file gpurun_out/mode_${tag}_${i}_$m.csv python scripts/prof_one.py $m > /dev/null 2>&1
  echo "$i: $setting" >> gpurun_out/mode_${tag}_settings.txt
  i=$((i+1))
done
