#!/bin/bash
# dW band per M side (current tree) vs HEAD (4 wide blocks everywhere): C1 bench alternating
for i in 1 2 3; do for lib in scripts/_bin/libsmoe_bandbase.so cur; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bab.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C1', round(d['value']), round(d['ms_per_step'],2), round(d['kernels']['group_xty']['ms_per_launch'],3))" gpurun_out/bab.log $lib
done; done
