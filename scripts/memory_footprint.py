"""GPU memory footprint: fused ScatterMoE path vs a padded group-copy baseline.

SURVEY.md §8f-4 / BASELINE "zero padding memory": reproduces the paper's
memory comparison (reference oracle.py:236-324) on B200.

  fused    : smoe_mlp_forward + smoe_mlp_backward (this package)
  padded   : the conventional staging the fused kernels avoid — copy tokens into
             per-expert groups padded to a block multiple (128), batched dense
             matmuls (torch.bmm, pad rows included), copy back, combine;
             autograd through it.

Reports peak allocated bytes above the resident inputs/weights for one
training step (forward + backward), and the padded rows the baseline carries.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402

BLOCK = 128


def padded_step(x, w1, w2, routing, order, dy):
    """Megablocks-style padded grouping, autograd for the backward."""
    t, k = routing.expert_idx.shape
    e, d, de = w1.shape
    counts = order.bin_counts.to(torch.int64)
    padded = ((counts + BLOCK - 1) // BLOCK) * BLOCK
    cap = int(padded.max())
    xg = torch.zeros((e, cap, d), dtype=x.dtype, device=x.device)
    pos = torch.arange(order.num_slots, device=x.device) - torch.repeat_interleave(order.bin_offsets[:-1].long(), counts)
    ex = torch.repeat_interleave(torch.arange(e, device=x.device), counts)
    xr = x.detach().requires_grad_(True)
    w1r, w2r = w1.detach().requires_grad_(True), w2.detach().requires_grad_(True)
    src = order.o.long() // k
    xg = xg.index_put((ex, pos), xr[src])                        # group copy (padded)
    h = torch.nn.functional.gelu(torch.bmm(xg, w1r))            # pad rows computed too
    yg = torch.bmm(h, w2r)
    y_slots = torch.empty((order.num_slots, d), dtype=x.dtype, device=x.device)
    y_slots = y_slots.index_put((order.o.long(),), yg[ex, pos])  # scatter back
    y = (routing.p.to(x.dtype).unsqueeze(-1) * y_slots.view(t, k, d)).sum(1)
    y.backward(dy)
    return int((padded - counts).sum()), int(padded.sum())


def fused_step(x, w1, w2, routing, order, dy):
    y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    sm.smoe_mlp_backward(ctx, dy)


def measure(fn, *args):
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    out = fn(*args)
    torch.cuda.synchronize()
    return torch.cuda.max_memory_allocated() - base, out


def main():
    rows = []
    for name, (t, d, de, e, k) in {"C1": (32768, 4096, 14336, 8, 2), "C2": (32768, 4096, 1792, 64, 8),
                                   "paper_E32_k4": (61440, 4096, 2048, 32, 4)}.items():
        g = torch.Generator(device="cuda").manual_seed(0)
        x = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        dy = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        w1 = ((torch.rand(e, d, de, device="cuda", generator=g) * 2 - 1) / d ** 0.5).bfloat16()
        w2 = ((torch.rand(e, de, d, device="cuda", generator=g) * 2 - 1) / de ** 0.5).bfloat16()
        routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
        order = sm.compute_grouped_order(routing)
        fused, _ = measure(fused_step, x, w1, w2, routing, order, dy)
        padded, (pad_rows, total_rows) = measure(padded_step, x, w1, w2, routing, order, dy)
        rows.append(dict(config=name, T=t, d_model=d, d_expert=de, E=e, k=k, fused_peak_gb=fused / 1e9,
                         padded_peak_gb=padded / 1e9, ratio=fused / padded, padded_rows=pad_rows,
                         padded_total_rows=total_rows, fused_padding_rows=0))
        print(json.dumps(rows[-1]), flush=True)
        del x, dy, w1, w2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
