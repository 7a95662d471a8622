#!/bin/bash
# Round-end evidence refresh on one B200: tests, smoke, bench lines (C1 with the
# CPU baseline, C2, reference arm, EP peer at N=1), C3, inference, memory, sort.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/rf_pytest.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/rf_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/rf_smoke.log
timeout 400 python bench.py > gpurun_out/rf_bench_c1.log 2>&1; echo "bench c1 rc $?"
timeout 400 python bench.py --config C2 > gpurun_out/rf_bench_c2.log 2>&1; echo "bench c2 rc $?"
timeout 300 python bench.py --impl reference > gpurun_out/rf_bench_ref.log 2>&1; echo "ref rc $?"
timeout 300 python bench.py --ep peer --no-cpu-baseline > gpurun_out/rf_bench_ep_peer.log 2>&1; echo "ep rc $?"
timeout 300 python scripts/momha_bench.py > gpurun_out/rf_c3.log 2>&1; echo "c3 rc $?"
timeout 300 python scripts/infer_bench.py C1 > gpurun_out/rf_inf_c1.log 2>&1; echo "inf rc $?"
timeout 300 python scripts/infer_bench.py C2 > gpurun_out/rf_inf_c2.log 2>&1
timeout 300 python scripts/memory_footprint.py > gpurun_out/rf_mem.log 2>&1; echo "mem rc $?"
timeout 300 python scripts/sort_bench.py > gpurun_out/rf_sort.log 2>&1; echo "sort rc $?"
for f in rf_bench_c1 rf_bench_c2 rf_bench_ref rf_bench_ep_peer; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'))" gpurun_out/$f.log
done
tail -c 400 gpurun_out/rf_c3.log; echo; tail -c 300 gpurun_out/rf_inf_c1.log; echo
