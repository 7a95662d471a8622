#!/bin/bash
# C1 / C2 bench: staged TMA-store epilogue on every grouped-output kernel (SMOE_TC_EPI=all) vs default
for i in 1 2 3; do for v in default all; do
  SMOE_TC_EPI=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ea_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C1 epi', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), {l[:26]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/ea_$v.log $v
done; done
for v in default all; do
  SMOE_TC_EPI=$v timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/ea2_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C2 epi', sys.argv[2], round(d['value']), round(d['ms_per_step'],2))" gpurun_out/ea2_$v.log $v
done
