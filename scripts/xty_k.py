"""group_xty efficiency vs bin length (tokens) — probes per-tile fixed overheads."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


d, de, E, k = 4096, 14336, 8, 2
for T in (4096, 8192, 16384, 32768, 65536):
    n = T * k
    g = torch.Generator(device="cuda").manual_seed(0)
    xg = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    h = (torch.rand(n, de, device="cuda", generator=g) * 2 - 1).bfloat16()
    routing = sm.topk_select(torch.softmax(torch.randn(T, E, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    fl = 2.0 * n * d * de
    t1 = timeit(lambda: sm.group_xty(xg, h, order))
    t2 = timeit(lambda: sm.scatter2scatter(xg, h.view(E, -1, de)[:, :d, :].contiguous() if False else
                                           torch.empty(0), order, 1) if False else None)
    print(f"T={T:6d} bin~{n // E:6d}  dW1 xty {t1:7.3f} ms {fl / t1 / 1e9:7.1f} TF/s", flush=True)
    del xg, h
