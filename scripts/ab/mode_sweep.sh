#!/bin/bash
# Base-clock ncu comparison of GEMM modes (tensor-pipe activity, DRAM, time).
# usage: mode_sweep.sh TAG mode...   (env vars pass through, e.g. SMOE_TC_CTAS=1)
tag=$1; shift
for m in "$@"; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -s 2 -c 1 --csv --log-file gpurun_out/mode_${tag}_$m.csv python scripts/prof_one.py $m > /dev/null 2>&1
done
