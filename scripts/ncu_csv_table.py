"""Per-launch table from an `ncu --metrics ... --csv` log: one row per kernel launch."""
import csv
import sys
from collections import OrderedDict


def launches(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"][:40])
        v = r["Metric Value"].replace(",", "")
        rows.setdefault(key, {})[r["Metric Name"] + " [" + r["Metric Unit"] + "]"] = float(v) if v else 0.0
    return rows


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(path)
        for (i, name), m in launches(path).items():
            print(" ", i, name, "  ".join(f"{k.split('.')[0][:28]}={v:.4g}" for k, v in sorted(m.items())))
