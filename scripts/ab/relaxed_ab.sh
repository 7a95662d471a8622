#!/bin/bash
# Relaxed ring_empty arrive (current tree) vs HEAD~ (release.cluster arrive): C3 o-proj GEMM, C3 projections, C1/C2 bench
B=scripts/_bin/libsmoe_base.so
timeout 600 python -m pytest tests/test_tcgen05_gpu.py tests/test_kernels_gpu.py tests/test_mlp_gpu.py tests/test_ep_peer.py -m gpu -q 2>&1 | tail -1
for lib in $B cur; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  SMOE_PROF_CFG=C3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm -c 1 --csv --log-file gpurun_out/ra_$(basename $lib).csv python scripts/prof_one.py ofwd > /dev/null 2>&1
  python scripts/ncu_csv_table.py gpurun_out/ra_$(basename $lib).csv | tail -1 | sed "s|^|$lib ofwd |"
done
for i in 1 2; do for lib in $B cur; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  timeout 300 python scripts/momha_bench.py > gpurun_out/ra_c3.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C3 proj', round(d['projections']['ms_per_step'],4), 'layer', round(d['layer']['ms_per_step'],3))" gpurun_out/ra_c3.log $lib
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ra_c1.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C1', round(d['value']), round(d['ms_per_step'],2))" gpurun_out/ra_c1.log $lib
  timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/ra_c2.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C2', round(d['value']), round(d['ms_per_step'],2))" gpurun_out/ra_c2.log $lib
done; done
