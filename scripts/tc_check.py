"""Quick tcgen05-vs-SIMT cross-check of every GEMM mode (debug aid; prints rel errors)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402


def rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def main(big=False):
    torch.manual_seed(0)
    dev = "cuda"
    cases = [(300, 2, 6, 256, 512), (1000, 2, 8, 128, 256), (77, 3, 5, 64, 192)]
    if big:
        cases.append((8192, 2, 8, 1024, 2048))
    for (T, k, E, d_in, d_out) in cases:
        ids = torch.stack([torch.randperm(E)[:k] for _ in range(T)]).to(dev)
        p = torch.rand(T, k, device=dev)
        routing = sm.RoutingResult(ids, p, torch.zeros(T, E, device=dev), renormalized=False, validate=False)
        order = sm.compute_grouped_order(routing)
        n = T * k
        xs = (torch.rand(T, d_in, device=dev) * 2 - 1).bfloat16()
        xg = (torch.rand(n, d_in, device=dev) * 2 - 1).bfloat16()
        w = ((torch.rand(E, d_in, d_out, device=dev) * 2 - 1) / d_in ** 0.5).bfloat16()
        wt = ((torch.rand(E, d_out, d_in, device=dev) * 2 - 1) / d_in ** 0.5).bfloat16()
        for name, x, lay, fan in (("S2G", xs, sm.SCATTERED_TO_GROUPED, k), ("S2S", xs, sm.SCATTERED_TO_SCATTERED, k),
                                  ("G2S", xg, sm.GROUPED_TO_SCATTERED, 1), ("G2G", xg, sm.GROUPED_TO_GROUPED, 1)):
            for tr, ww in ((False, w), (True, wt)):
                a = sm.scatter2scatter(x, ww, order, fan, lay, transpose_w=tr, engine="simt")
                b = sm.scatter2scatter(x, ww, order, fan, lay, transpose_w=tr, engine="tcgen05")
                torch.cuda.synchronize()
                print(f"T={T} E={E} {d_in}x{d_out} {name} trans={tr}: rel={rel(b, a):.3e}", flush=True)
        yg = (torch.rand(n, d_out, device=dev) * 2 - 1).bfloat16()
        a = sm.group_xty(xg, yg, order, engine="simt")
        b = sm.group_xty(xg, yg, order, engine="tcgen05")
        torch.cuda.synchronize()
        print(f"T={T} E={E} group_xty {d_in}x{d_out}: rel={rel(b, a):.3e}", flush=True)
        pre_a = torch.empty(n, d_out, device=dev, dtype=torch.bfloat16); h_a = torch.empty_like(pre_a)
        pre_b = torch.empty_like(pre_a); h_b = torch.empty_like(pre_a)
        sm.scatter2scatter(xs, w, order, k, sm.SCATTERED_TO_GROUPED, out=pre_a, activation="gelu", act_out=h_a, engine="simt")
        sm.scatter2scatter(xs, w, order, k, sm.SCATTERED_TO_GROUPED, out=pre_b, activation="gelu", act_out=h_b, engine="tcgen05")
        torch.cuda.synchronize()
        print(f"  act epilogue: pre {rel(pre_b, pre_a):.3e} h {rel(h_b, h_a):.3e}", flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main(big="big" in sys.argv)
    print("done", time.time() - t0)
