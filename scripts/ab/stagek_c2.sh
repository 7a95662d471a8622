#!/bin/bash
# C2: staged (coalesced / TMA-store) epilogue for the K = 1792 GEMMs vs direct stores
for i in 1 2; do for s in 1024 2048; do
  SMOE_TC_STAGE_K=$s timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/sk_$s.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C2 stage_k', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), {l[:26]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/sk_$s.log $s
done; done
