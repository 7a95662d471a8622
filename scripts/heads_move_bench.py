"""Slot rows <-> attention heads moves at C3 (n = 131072 slot rows of 512 bf16): us per call."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402

b, seq, k, h, dh, e = 8, 4096, 4, 4, 128, 16
t = b * seq
g = torch.Generator(device="cuda").manual_seed(0)
routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
order = sm.compute_grouped_order(routing)
rows = torch.randn(t * k, h * dh, device="cuda", generator=g).bfloat16()
heads = sm.kernels.grouped_to_heads(rows, order, k, b, seq, dh)


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def permute_copy():
    return rows.view(b, seq, k, h, dh).permute(0, 3, 2, 1, 4).contiguous()


print(json.dumps({"grouped_to_heads_us": timeit(lambda: sm.kernels.grouped_to_heads(rows, order, k, b, seq, dh)),
                  "heads_to_grouped_us": timeit(lambda: sm.kernels.heads_to_grouped(heads, order, k)),
                  "torch_permute_copy_us": timeit(permute_copy),
                  "bytes_moved": 2 * rows.numel() * 2}))
