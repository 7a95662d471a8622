#!/bin/bash
# C2: dW1 with X gathered by slot (no grouped copy) vs group() + TMA-fed dW1
for i in 1 2; do for g in 1024 2048; do
  SMOE_GATHER_MAX_DOUT=$g timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/gc2_$g.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C2 gather_max_dout', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), {l[:24]: round(v['ms_per_launch'],3) for l,v in k.items() if 'xty' in l or l=='group'})" gpurun_out/gc2_$g.log $g
done; done
