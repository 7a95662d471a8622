#!/bin/bash
# Wide-tile policy A/B: GPU tests at the default policy, then C1 bench and C3
# projections alternating SMOE_TC_WIDE=0 and the default.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w2_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/w2_pytest.log
for i in 1 2 3; do for w in 0 d; do
  if [ $w = 0 ]; then export SMOE_TC_WIDE=0; else unset SMOE_TC_WIDE; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/w2_bench_$w.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C1 wide', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {l: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/w2_bench_$w.log $w
done; done
unset SMOE_TC_WIDE
for w in 0 d; do
  if [ $w = 0 ]; then export SMOE_TC_WIDE=0; else unset SMOE_TC_WIDE; fi
  timeout 300 python scripts/momha_bench.py > gpurun_out/w2_c3_$w.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C3 wide', sys.argv[2], d['projections']['ms_per_step'], d['layer']['ms_per_step'])" gpurun_out/w2_c3_$w.log $w
done
