#!/bin/bash
# Staged epilogue for scattered-output kernels: C2 bench and C3 projections, A/B alternating
for i in 1 2; do for v in 0 1; do
  SMOE_TC_STAGE_SCATTERED=$v timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/ss_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C2 stage_scattered', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), {l[:26]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/ss_$v.log $v
  SMOE_TC_STAGE_SCATTERED=$v timeout 300 python scripts/momha_bench.py > gpurun_out/ss_c3_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C3 stage_scattered', sys.argv[2], round(d['projections']['ms_per_step'],4))" gpurun_out/ss_c3_$v.log $v
done; done
for v in 0 1; do
  SMOE_TC_STAGE_SCATTERED=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ss1_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C1 stage_scattered', sys.argv[2], round(d['value']), round(d['ms_per_step'],2))" gpurun_out/ss1_$v.log $v
done
