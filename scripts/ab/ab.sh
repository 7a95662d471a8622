#!/bin/bash
# Interleaved base-clock ncu A/B of GEMM modes across library builds in one session.
# usage: ab.sh TAG "variant1 variant2 ..." mode...   (variant "cur" = in-tree build,
# others = scripts/_bin/libsmoe_<variant>.so from build_variant.sh)
tag=$1; variants=$2; shift 2
for m in "$@"; do
  for v in $variants; do
    if [ "$v" = cur ]; then lib=""; else lib="$PWD/scripts/_bin/libsmoe_$v.so"; fi
    SMOE_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -s 2 -c 1 --csv --log-file gpurun_out/mode_${tag}_${v}_$m.csv python scripts/prof_one.py $m > /dev/null 2>&1
  done
done
