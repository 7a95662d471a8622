"""Per-call device timing of the library's kernels (measurement aid for bench.py).

While a ``LaunchTimer`` is active, every C-ABI call made through this package
(`kernels.py`, the routing sort in `router.py`) is bracketed by two CUDA
events recorded on the stream the kernel is launched on, under a label that
names the call and its mode (e.g. ``scatter2scatter S->G +act``).  After the
region, ``summary()`` synchronises and returns per-label launch counts and
mean device durations.  Nothing is recorded when no timer is active, so the
normal path (and CUDA-graph capture) is untouched.
"""
from __future__ import annotations

from collections import OrderedDict

import torch

_active: "LaunchTimer | None" = None


class LaunchTimer:
    def __init__(self):
        self.records: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def __enter__(self) -> "LaunchTimer":
        global _active
        if _active is not None:
            raise RuntimeError("a LaunchTimer is already active")
        _active = self
        return self

    def __exit__(self, *exc) -> None:
        global _active
        _active = None

    def summary(self) -> "OrderedDict[str, dict]":
        """{label: {"launches": n, "ms_total": t, "ms_per_launch": t/n}} in first-seen order."""
        torch.cuda.synchronize()
        out: "OrderedDict[str, dict]" = OrderedDict()
        for label, e0, e1 in self.records:
            d = out.setdefault(label, {"launches": 0, "ms_total": 0.0})
            d["launches"] += 1
            d["ms_total"] += e0.elapsed_time(e1)
        for d in out.values():
            d["ms_per_launch"] = d["ms_total"] / d["launches"]
        return out


def begin(stream: torch.cuda.Stream | None = None):
    """Start event for one library call, or None when no timer is active."""
    if _active is None:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def end(label: str, start, stream: torch.cuda.Stream | None = None) -> None:
    if start is None or _active is None:
        return
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    _active.records.append((label, start, e))
