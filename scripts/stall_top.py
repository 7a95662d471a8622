"""Top stall-sampled SASS instructions of an ncu source-page CSV export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[wi]), r[ai][-5:], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for w, a, s in sorted(data, reverse=True)[:n]:
    print(f"{w:8d} {100 * w / tot:5.1f}% {a} {s[:100]}")
