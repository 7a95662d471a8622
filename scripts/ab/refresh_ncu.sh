#!/bin/bash
# ncu evidence for the round: launch list of one C1 bench step, and one
# --set full capture per C1 GEMM mode (DRAM traffic -> profiles/traffic.json).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rn_launches_c1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rn_bench_under_ncu.log 2>&1; echo "launches rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rn_launches_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches c2 rc $?"
for m in xty l1s dhs l2 dx; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc2_gemm -c 1 -o gpurun_out/rn_full_$m python scripts/prof_one.py $m > /dev/null 2>&1; echo "full $m rc $?"
done
# keep the merge-back small: raw pages as CSV, reports deleted
for m in xty l1s dhs l2 dx; do
  ncu -i gpurun_out/rn_full_$m.ncu-rep --page raw --csv > gpurun_out/rn_full_$m.csv 2>/dev/null
  ncu -i gpurun_out/rn_full_$m.ncu-rep --page source --csv --print-source sass > gpurun_out/rn_sass_$m.csv 2>/dev/null
  rm -f gpurun_out/rn_full_$m.ncu-rep
done
gzip -f gpurun_out/rn_sass_*.csv
du -sh gpurun_out
