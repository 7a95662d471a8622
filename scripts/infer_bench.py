"""Inference forward (smoe_mlp_forward(training=False)) timing on one B200.

The inference path is the reference's scatter_combine route (kernels.py:242-286,
parallel_linear.py:120-126): layer 1 S->G with the activation fused (no
pre-activation kept), layer 2 as scatter_combine (bf16: a scattered-output
GEMM + the token-major combine; SMOE_COMBINE_FUSED=1 reduces the p-scaled
rows into fp32 token rows in the GEMM epilogue instead).  FLOPs per forward
= 4*T*k*d*d_e.  Prints one JSON line with per-kernel times (launch_timer).
usage: python scripts/infer_bench.py [C1|C2] [engine]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402
from paper_2403_08245_b200.launch_timer import LaunchTimer  # noqa: E402

CFG = {"C1": (32768, 4096, 14336, 8, 2), "C2": (32768, 4096, 1792, 64, 8)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    if len(sys.argv) > 2:
        sm.set_engine(sys.argv[2])
    T, d, de, E, k = CFG[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand((T, d), generator=g, device="cuda") * 2 - 1).bfloat16()
    w1 = ((torch.rand((E, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).bfloat16()
    w2 = ((torch.rand((E, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).bfloat16()
    wg = (torch.rand((d, E), generator=g, device="cuda") * 2 - 1) / d ** 0.5
    routing = sm.topk_select(sm.gate_forward(x.float(), wg), k)

    def step():
        order = sm.compute_grouped_order(routing)
        return sm.smoe_mlp_forward(x, w1, w2, routing, order, training=False)[0]

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    steps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    with LaunchTimer() as lt:
        for _ in range(steps):
            step()
    kern = {lab: {"ms_per_launch": v["ms_per_launch"], "launches_per_step": v["launches"] / steps}
            for lab, v in lt.summary().items()}
    flops = 4.0 * T * k * d * de
    print(json.dumps({"workload": f"{name} inference forward T={T} d={d} d_e={de} E={E} k={k}",
                      "engine": sm.get_engine(), "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
                      "tflops": flops / (ms / 1e3) / 1e12, "kernels": kern,
                      "peak_memory_gb": torch.cuda.max_memory_allocated() / 1e9}))


if __name__ == "__main__":
    main()
