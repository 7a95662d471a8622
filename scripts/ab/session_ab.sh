#!/bin/bash
# This session's engine changes (current tree) vs the session-start library (315df6e), alternating on one box.
# (Python-side changes — the MoMHA path — are current in both arms; only libsmoe_b200.so differs.)
for i in 1 2 3; do for lib in scripts/_bin/libsmoe_start.so cur; do
  if [ $lib = cur ]; then unset SMOE_LIB SMOE_LIB_ALLOW_MISSING; else export SMOE_LIB=$lib SMOE_LIB_ALLOW_MISSING=1; fi
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/sa_c1.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C1', round(d['value']), round(d['ms_per_step'],2))" gpurun_out/sa_c1.log $lib
done; done
for lib in scripts/_bin/libsmoe_start.so cur; do
  if [ $lib = cur ]; then unset SMOE_LIB SMOE_LIB_ALLOW_MISSING; else export SMOE_LIB=$lib SMOE_LIB_ALLOW_MISSING=1; fi
  timeout 300 python bench.py --no-cpu-baseline --config C2 --steps 20 > gpurun_out/sa_c2.log 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'C2', round(d['value']), round(d['ms_per_step'],2))" gpurun_out/sa_c2.log $lib
done
