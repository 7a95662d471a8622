#!/bin/bash
# act-grad operand prefetch in the staged epilogue: parity, C3 projections, wide dH waits, C1 bench
timeout 600 python -m pytest tests/test_tcgen05_gpu.py tests/test_parallel_linear_gpu.py tests/test_mlp_gpu.py -m gpu -q 2>&1 | tail -2
timeout 300 python scripts/momha_bench.py > gpurun_out/ap_c3.log 2>&1
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C3', d['projections']['ms_per_step'], {k: round(v['ms_per_launch'],3) for k,v in d['projections']['kernels'].items()})" gpurun_out/ap_c3.log
for m in dhs l1s; do echo "== $m wide forced"; SMOE_TC_WIDE=1 SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py $m 2>&1 | grep "timing cluster" | tail -2; done
echo "== dhs default"; SMOE_TC_TIMING=1 timeout 120 python scripts/prof_one.py dhs 2>&1 | grep "timing cluster" | tail -1
