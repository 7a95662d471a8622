#!/bin/bash
# Alternating full-step A/B of library builds on one box (the power-capped step
# varies +-3 % box to box, so only same-box alternation is meaningful).
# usage: step_ab.sh ROUNDS "lib1 lib2 ..." [bench args]   (lib "cur" = in-tree build,
# others = scripts/_bin/libsmoe_<lib>.so); prints one summary line per run.
rounds=$1; libs=$2; shift 2
for r in $(seq 1 "$rounds"); do
  for v in $libs; do
    if [ "$v" = cur ]; then lib=""; else lib="$PWD/scripts/_bin/libsmoe_$v.so"; fi
    SMOE_LIB=$lib SMOE_LIB_ALLOW_MISSING=1 timeout 600 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v', 'r$r', round(d['value']), 'ms', round(d['ms_per_step'],3), 'med', round(d['step_ms']['median'],3), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'), ' '.join(f\"{l.split(' ')[0][:5]}{l[15:24].strip()}={v['ms_per_launch']:.3f}\" for l, v in k.items() if v['ms_per_launch'] > 1))"
  done
done
