for h in off keep keepfirst; do
  for m in l2 dx xty rows; do
    SMOE_L2_HINT=$h timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:gemm -s 2 -c 1 --csv python scripts/prof_one.py $m 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v h=$h -v m=$m '{print h, m, $(NF-2), $NF}'
  done
done
for h in off keep keepfirst off keep keepfirst; do echo "== $h"; SMOE_L2_HINT=$h timeout 300 python scripts/energy.py l2 xty dx rows 2>&1 | grep -v Warn; done
