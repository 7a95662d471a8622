#!/bin/bash
# C2 (bins of 4096 rows, K = 1792 / 4096): wide-tile thresholds
for i in 1 2; do for v in d b bk; do
  unset SMOE_TC_WIDE_MIN_BIN SMOE_TC_WIDE_MIN_K
  [ $v = b ] && export SMOE_TC_WIDE_MIN_BIN=2048
  [ $v = bk ] && export SMOE_TC_WIDE_MIN_BIN=2048 SMOE_TC_WIDE_MIN_K=1024
  timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/wc2_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C2', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {l[:22]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/wc2_$v.log $v
done; done
