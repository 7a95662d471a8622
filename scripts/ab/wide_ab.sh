#!/bin/bash
# Wide (512-row) vs 256-row pair tiles: parity tests with wide tiles forced,
# energy per launch of each TMA-fed C1 GEMM, and the C1/C2 bench step.
mkdir -p gpurun_out
SMOE_TC_WIDE=1 timeout 600 python -m pytest tests/test_tcgen05_gpu.py tests/test_kernels_gpu.py tests/test_mlp_gpu.py -m gpu -x -q > gpurun_out/w_pytest_forced.log 2>&1; echo "pytest (wide forced) rc $?"; tail -2 gpurun_out/w_pytest_forced.log
for w in 0 1; do SMOE_TC_WIDE=$w timeout 200 python scripts/energy.py rows xty l2 dh dx > gpurun_out/w_energy_$w.jsonl 2>&1; done
for w in 0 1 0 1; do SMOE_TC_WIDE=$w timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/w_bench_$w.log 2>&1; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('wide', sys.argv[2], d['value'], d['ms_per_step'], d['clocks'])" gpurun_out/w_bench_$w.log $w; done
for w in 0 1; do SMOE_TC_WIDE=$w timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/w_bench_c2_$w.log 2>&1; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('C2 wide', sys.argv[2], d['value'], d['ms_per_step'])" gpurun_out/w_bench_c2_$w.log $w; done
cat gpurun_out/w_energy_0.jsonl gpurun_out/w_energy_1.jsonl
