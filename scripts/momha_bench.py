"""C3 mixture-of-attention timing on one B200 (BASELINE.json configs[3]).

E=16, k=4, d_model=2048, d_head=128, 4 heads per expert (d_proj=512), 16
active heads, B=8 sequences of 4096 tokens (T=32768), causal, bf16.

Reports, with CUDA events after warm-up (inputs resident in HBM):
  * the routed projections alone (ParallelLinear q: S->S fan-out 4, o: S->S with
    the gate combine; forward + backward) in tokens/s and TFLOP/s, FLOPs
    12*T*k*d_model*d_proj (the hot path);
  * the whole MoMHA layer step (projections + shared K/V GEMMs + fused SDPA core).
Prints one JSON line.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402
import importlib  # noqa: E402

pl = importlib.import_module("paper_2403_08245_b200.parallel_linear")  # the module (the package re-exports a function)


def timed(fn, steps=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    b, seq, e, k, d, dh, hpe = 8, 4096, 16, 4, 2048, 128, 4
    t = b * seq
    cfg = sm.MomhaConfig(d_model=d, d_head=dh, num_heads=k * hpe, heads_per_expert=hpe, num_experts=e, k=k)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand((t, d), device="cuda", generator=g) * 2 - 1).bfloat16()
    dy = (torch.rand((t, d), device="cuda", generator=g) * 2 - 1).bfloat16()
    wts = sm.init_momha_weights(cfg, 0, dtype=torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    dp_ = cfg.d_proj
    attn = (torch.rand((t * k, dp_), device="cuda", generator=g) * 2 - 1).bfloat16()
    dq = (torch.rand((t * k, dp_), device="cuda", generator=g) * 2 - 1).bfloat16()

    def projections():
        q, qc = pl.forward(x, wts.wq, order, p=None, fan_out=k, layout=sm.SCATTERED_TO_SCATTERED)
        y, oc = pl.forward(attn, wts.wo, order, p=routing.p, fan_out=1, layout=sm.SCATTERED_TO_SCATTERED)
        pl.backward(oc, dy)
        pl.backward(qc, dq)

    def layer():
        y, ctx = sm.momha_forward(x, wts, routing, order, cfg, seq)
        sm.momha_backward(ctx, dy)

    ms_proj = timed(projections)
    from paper_2403_08245_b200.launch_timer import LaunchTimer
    with LaunchTimer() as lt:
        for _ in range(5):
            projections()
    kern = {lab: {"ms_per_launch": v["ms_per_launch"], "launches_per_step": v["launches"] / 5}
            for lab, v in lt.summary().items()}
    ms_layer = timed(layer, steps=20, warmup=3)
    flops = 12.0 * t * k * d * dp_
    line = {
        "workload": "C3 MoMHA: B=8 x seq 4096 (T=32768), E=16, k=4, d_model=2048, d_head=128, d_proj=512, causal, bf16",
        "projections": {"ms_per_step": ms_proj, "tokens_per_s": t / (ms_proj / 1e3),
                        "tflops": flops / (ms_proj / 1e3) / 1e12, "flop_per_step": flops,
                        "what": "ParallelLinear q (S->S, fan-out 4) + o (S->S, gate combine), fwd+bwd",
                        "kernels": kern},
        "layer": {"ms_per_step": ms_layer, "tokens_per_s": t / (ms_layer / 1e3),
                  "what": "momha_forward + momha_backward (projections, shared K/V GEMMs, fused SDPA core)"},
        "launches_note": "projection kernels from libsmoe_b200.so; K/V GEMMs and SDPA are torch library kernels",
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
