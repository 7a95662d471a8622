"""Time each tcgen05 GEMM variant at C1 shapes with CUDA events (perf triage)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    T, d, de, E, k = 32768, 4096, 14336, 8, 2
    if len(sys.argv) > 1 and sys.argv[1] == "C2":
        T, d, de, E, k = 32768, 4096, 1792, 64, 8
    n = T * k
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    x = (torch.rand(T, d, device=dev, generator=g) * 2 - 1).bfloat16()
    xg = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).bfloat16()
    w1 = ((torch.rand(E, d, de, device=dev, generator=g) * 2 - 1) / d ** 0.5).bfloat16()
    w2 = ((torch.rand(E, de, d, device=dev, generator=g) * 2 - 1) / de ** 0.5).bfloat16()
    logits = torch.randn(T, E, device=dev, generator=g)
    routing = sm.topk_select(torch.softmax(logits, 1), k)
    order = sm.compute_grouped_order(routing)
    h = torch.empty(n, de, device=dev, dtype=torch.bfloat16)
    h2 = torch.empty_like(h)
    y = torch.empty(n, d, device=dev, dtype=torch.bfloat16)
    fl = 2.0 * n * d * de
    res = {}
    res["L1 S2G gather, epi none"] = timeit(lambda: sm.scatter2scatter(x, w1, order, k, sm.SCATTERED_TO_GROUPED, out=h))
    res["L1 S2G gather, act (pre+h)"] = timeit(lambda: sm.scatter2scatter(x, w1, order, k, sm.SCATTERED_TO_GROUPED, out=h, activation="gelu", act_out=h2))
    res["L1 S2G gather, act only"] = timeit(lambda: sm.scatter2scatter(x, w1, order, k, sm.SCATTERED_TO_GROUPED, out=h, activation="gelu"))
    res["L1 S2G gather, relu (pre+h)"] = timeit(lambda: sm.scatter2scatter(x, w1, order, k, sm.SCATTERED_TO_GROUPED, out=h, activation="relu", act_out=h2))
    res["L1-shape G2G rows, epi none"] = timeit(lambda: sm.scatter2scatter(xg, w1, order, 1, sm.GROUPED_TO_GROUPED, out=h))
    res["L2 G2S rows (K=de)"] = timeit(lambda: sm.scatter2scatter(h, w2, order, 1, sm.GROUPED_TO_SCATTERED, out=y))
    res["dH G2G W2^T, none"] = timeit(lambda: sm.scatter2scatter(xg, w2, order, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, out=h2))
    res["dH G2G W2^T, act_grad"] = timeit(lambda: sm.scatter2scatter(xg, w2, order, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, out=h2, activation="gelu", act_grad_of=h))
    res["dX G2S W1^T (K=de)"] = timeit(lambda: sm.scatter2scatter(h, w1, order, 1, sm.GROUPED_TO_SCATTERED, transpose_w=True, out=y))
    res["dW2 xty H^T dY"] = timeit(lambda: sm.group_xty(h, xg, order))
    res["dW1 xty X^T dH"] = timeit(lambda: sm.group_xty(xg, h, order))
    for kk, v in res.items():
        print(f"{kk:34s} {v:8.3f} ms  {fl / v / 1e9:8.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
