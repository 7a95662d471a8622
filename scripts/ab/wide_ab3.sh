#!/bin/bash
# C1 bench: wide tiles off / grouped-K only / grouped-K + K>=8192 grouped-M (default)
for i in 1 2 3; do for w in 0 x d; do
  unset SMOE_TC_WIDE SMOE_TC_WIDE_MIN_K
  [ $w = 0 ] && export SMOE_TC_WIDE=0
  [ $w = x ] && export SMOE_TC_WIDE_MIN_K=1000000000
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/w3_bench_$w.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C1 wide', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {l[:18]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/w3_bench_$w.log $w
done; done
