#!/bin/bash
# Gather cp.async L2 prefetch hint: 256 B (default build) vs 128 B vs none: C1 layer-1 GEMM alone and the C1 step
for lib in cur scripts/_bin/libsmoe_hint128.so scripts/_bin/libsmoe_hint0.so; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/gh_$(basename $lib).csv python scripts/prof_one.py l1s > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/gh_$(basename $lib).csv | tail -1 | sed "s|^|$lib |" | cut -c 1-250
done
for i in 1 2; do for lib in cur scripts/_bin/libsmoe_hint128.so scripts/_bin/libsmoe_hint0.so; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/gh_c1.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print(sys.argv[2], 'C1', round(d['value']), round(d['ms_per_step'],2), round(k['scatter2scatter S->G +act(pre,post) scaled']['ms_per_launch'],3))" gpurun_out/gh_c1.log $lib
done; done
