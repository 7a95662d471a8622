#!/bin/bash
# Row kernels with the column loop unrolled by 4 (current tree) vs HEAD: C2 / C3 per-kernel times
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_mlp_gpu.py tests/test_momha_gpu.py -m gpu -q 2>&1 | tail -1
for i in 1 2; do for lib in scripts/_bin/libsmoe_rowbase.so cur; do
  if [ $lib = cur ]; then unset SMOE_LIB; else export SMOE_LIB=$lib; fi
  timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/ro_c2.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernels']; print(sys.argv[2], 'C2', round(d['value']), {l[:14]: round(v['ms_per_launch'],4) for l,v in k.items() if v['ms_per_launch']<1})" gpurun_out/ro_c2.log $lib
  timeout 300 python scripts/momha_bench.py > gpurun_out/ro_c3.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['projections']['kernels']; print(sys.argv[2], 'C3', round(d['projections']['ms_per_step'],4), {l[:14]: round(v['ms_per_launch'],4) for l,v in k.items() if v['ms_per_launch']<0.15})" gpurun_out/ro_c3.log $lib
done; done
