"""Summarise an ncu --metrics gpu__time_duration.sum launch list (our kernels only)."""
import csv
import re
import sys


def main(path, only_ours=True):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        if only_ours and "smoe" not in name and "gemm_kernel" not in name:
            continue
        short = re.sub(r"\(.*", "", name)
        m = re.search(r"(tc2?)_gemm_kernel<(\d+), (\d+), (\w+)(?:, (\w+))?(?:, (\w+))?>", name)
        if m:
            short = f"{m.group(1)}_gemm<A{m.group(2)},B{m.group(3)},GK={m.group(4)}"
            if m.group(5) is not None:
                short += f",STAGED={m.group(5)}"
            if m.group(6) is not None:
                short += f",WIDE={m.group(6)}"
            short += ">"
        out.append((int(r[ii]), short, float(r[vi].replace(",", "")) / 1e3))
    for i, s, us in out:
        print(f"{i:5d} {us:10.1f} us  {s}")
    return out


if __name__ == "__main__":
    main(sys.argv[1])
