"""Routing-sort kernel (K1, smoe_route_sort) timing and HBM bandwidth on one B200.

SURVEY.md §8(d): report the sort in µs and GB/s, at the bench configs' slot
counts (C1 n=65,536; C2 n=262,144) and at large n where bandwidth is
meaningful.  Algorithmic bytes per slot: int64 expert id in (8) + three int32
outputs (sorted_scattered_idxs, sorted_expert_idxs, inverse: 12) = 20 B.
Buffers are preallocated; the timed region is the C-ABI call alone (hist ->
scan -> scatter kernels), CUDA events, after warm-up.  One JSON line per n.
"""
import ctypes
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2403_08245_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())
    cases = ((65536, 8), (262144, 64), (1 << 24, 64), (1 << 26, 64))
    if len(sys.argv) > 1:  # e.g. `sort_bench.py 16777216:64` (profiling one size)
        cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
    for n, e in cases:
        ids = torch.randint(0, e, (n,), device="cuda", dtype=torch.int64)
        o = torch.empty(n, dtype=torch.int32, device="cuda")
        sid = torch.empty_like(o)
        inv = torch.empty_like(o)
        off = torch.empty(e + 1, dtype=torch.int32, device="cuda")
        wsb = lib.smoe_route_sort_workspace_bytes(n, e)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def call():
            rc = lib.smoe_route_sort(ids.data_ptr(), n, e, o.data_ptr(), sid.data_ptr(), off.data_ptr(),
                                     inv.data_ptr(), ws.data_ptr(), wsb, st)
            assert rc == 0, _lib.last_error()

        for _ in range(5):
            call()
        torch.cuda.synchronize()
        reps = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        # spot check: stable order, bit-exact vs torch's stable argsort
        if n <= 1 << 24:
            ref = torch.sort(ids, stable=True).indices.to(torch.int32)
            assert torch.equal(ref, o), "sort mismatch"
        gbs = 20.0 * n / (us * 1e-6) / 1e9
        print(json.dumps({"n": n, "E": e, "onepass_enabled": os.environ.get("SMOE_SORT_ONEPASS", "1") != "0", "us": us, "algorithmic_bytes": 20 * n, "GBps": gbs,
                          "frac_hbm": gbs / peaks["hbm_gbs"], "peak_hbm_gbs": peaks["hbm_gbs"]}), flush=True)


if __name__ == "__main__":
    main()
