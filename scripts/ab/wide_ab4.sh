#!/bin/bash
# Grouped wide-tile issue (first/last MMA groups of SMOE_TC_WIDE_DEFER stages):
# parity with wide tiles forced, issue-loop counters, and C1 bench per defer depth.
mkdir -p gpurun_out
SMOE_TC_WIDE=1 timeout 600 python -m pytest tests/test_tcgen05_gpu.py tests/test_kernels_gpu.py tests/test_mlp_gpu.py tests/test_parallel_linear_gpu.py -m gpu -x -q > gpurun_out/w4_pytest_forced.log 2>&1; echo "pytest (wide forced) rc $?"; tail -2 gpurun_out/w4_pytest_forced.log
for m in rows dh l2 xty; do for d in 1 4; do
  echo "== $m wide defer=$d"; SMOE_TC_WIDE=1 SMOE_TC_WIDE_DEFER=$d SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py $m 2>&1 | grep "timing cluster" | tail -2
done; done
for i in 1 2; do for d in 0 1 2 4; do
  unset SMOE_TC_WIDE; export SMOE_TC_WIDE_DEFER=$d; [ $d = 0 ] && export SMOE_TC_WIDE=0
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/w4_bench_$d.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print('C1 defer', sys.argv[2], round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {l[:22]: round(v['ms_per_launch'],3) for l,v in k.items() if v['ms_per_launch']>1})" gpurun_out/w4_bench_$d.log $d
done; done
