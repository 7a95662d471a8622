#!/bin/bash
# A/B of gathered backward operands (SMOE_GATHER_OPERANDS=1) vs grouped copies (=0)
# on C1, C2 (bench.py) and C3 (momha_bench.py); twice each, interleaved.
for rep in 1 2; do
  for g in 0 1; do
    SMOE_GATHER_MAX_DOUT=${MAXD:-1024} SMOE_GATHER_OPERANDS=$g timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/ab_c1_g${g}_$rep.log 2>&1
    SMOE_GATHER_MAX_DOUT=${MAXD:-1024} SMOE_GATHER_OPERANDS=$g timeout 300 python bench.py --config C2 --no-cpu-baseline > gpurun_out/ab_c2_g${g}_$rep.log 2>&1
    SMOE_GATHER_MAX_DOUT=${MAXD:-1024} SMOE_GATHER_OPERANDS=$g timeout 300 python scripts/momha_bench.py > gpurun_out/ab_c3_g${g}_$rep.log 2>&1
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_*.log")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    if "projections" in d:
        print(f, round(d["projections"]["ms_per_step"], 3))
    else:
        k = {n: round(v["ms_per_launch"], 3) for n, v in d["kernels"].items() if "xty" in n or n == "group"}
        print(f, round(d["ms_per_step"], 3), d["clocks"]["sm_mhz"], k)
PY
