import csv, sys
for m in sys.argv[1:]:
    rows = list(csv.reader(open(f"gpurun_out/mode_{m}.csv")))  # m may include a TAG_ prefix
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]; mi = h.index("Metric Name"); vi = h.index("Metric Value")
    d = {r[mi]: float(r[vi].replace(",", "")) for r in rows[hi + 1:] if len(r) > vi}
    t = d["gpu__time_duration.sum"] / 1e6
    print(f"{m:8s} t={t:6.3f}ms  tensor={d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:5.1f}%  "
          f"dram r/w={d['dram__bytes_read.sum']/1e9:5.2f}/{d['dram__bytes_write.sum']/1e9:5.2f} GB  clk={d['sm__cycles_elapsed.avg.per_second']/1e9:.2f}GHz")
