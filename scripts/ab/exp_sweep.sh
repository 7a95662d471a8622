#!/bin/bash
# usage: exp_sweep.sh TAG script [args]  — base-clock ncu of the 3rd gemm launch
tag=$1; shift
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -s 2 -c 1 --csv --log-file gpurun_out/mode_${tag}.csv python "$@" > /dev/null 2>&1
