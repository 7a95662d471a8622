"""Probe: is the 1-GPU training step CUDA-graph capturable, and what does replay save?"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402

T, d, de, E, k = 32768, 4096, 14336, 8, 2
if len(sys.argv) > 1 and sys.argv[1] == "C2":
    T, d, de, E, k = 32768, 4096, 1792, 64, 8
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = (torch.rand((T, d), generator=g, device=dev) * 2 - 1).bfloat16()
dy = (torch.rand((T, d), generator=g, device=dev) * 2 - 1).bfloat16()
cfg = sm.SmoeMlpConfig(d_model=d, d_expert=de, num_experts=E, k=k)
w1, w2 = sm.init_smoe_mlp_weights(cfg, 101, dtype=torch.bfloat16, device=dev, source="device")
wg = (torch.rand((d, E), generator=g, device=dev) * 2 - 1) / d ** 0.5
routing = sm.topk_select(sm.gate_forward(x.float(), wg), k)


def step():
    order = sm.compute_grouped_order(routing)
    y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    return y, sm.smoe_mlp_backward(ctx, dy)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


eager = timed(step)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        step()
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    out = step()
graph_ms = timed(graph.replay)
y_ref, g_ref = step()
graph.replay()
torch.cuda.synchronize()
same = torch.equal(out[0], y_ref) and torch.equal(out[1].dx, g_ref.dx) and torch.equal(out[1].dw1, g_ref.dw1)
print({"eager_ms": eager, "graph_ms": graph_ms, "bit_identical": same})
