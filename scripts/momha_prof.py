"""Kernel breakdown of one C3 MoMHA layer step (torch.profiler, CUDA time per kernel)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402


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

    def layer():
        y, ctx = sm.momha_forward(x, wts, routing, order, cfg, seq)
        sm.momha_backward(ctx, dy)

    for _ in range(3):
        layer()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        layer()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))


if __name__ == "__main__":
    main()
