"""Run one GEMM variant a few times (target for ncu -k regex:tc_gemm)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402

which = sys.argv[1]
import os  # noqa: E402
# SMOE_PROF_CFG=C2: the fine-grained config (E=64, k=8, d_expert=1792); default C1
# SMOE_PROF_CFG=C3: the MoMHA projections (d_model=2048, d_proj=512, E=16, k=4)
_CFGS = {"C2": (32768, 4096, 1792, 64, 8), "C3": (32768, 2048, 512, 16, 4)}
T, d, de, E, k = _CFGS.get(os.environ.get("SMOE_PROF_CFG", ""), (32768, 4096, 14336, 8, 2))
n = T * k
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = (torch.rand(T, d, device=dev, generator=g) * 2 - 1).bfloat16()
xg = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).bfloat16()
w = ((torch.rand(E, d, de, device=dev, generator=g) * 2 - 1) / d ** 0.5).bfloat16()
routing = sm.topk_select(torch.softmax(torch.randn(T, E, device=dev, generator=g), 1), k)
order = sm.compute_grouped_order(routing)
# operands with realistic values (uninitialised memory can hold NaN/Inf/denormal
# patterns that change the tensor pipe's behaviour); SMOE_PROF_EMPTY=1 keeps the old behaviour
import os  # noqa: E402
if os.environ.get("SMOE_PROF_EMPTY"):
    h = torch.empty(n, de, device=dev, dtype=torch.bfloat16)
else:
    h = ((torch.rand(n, de, device=dev, generator=g) * 2 - 1) * 0.5).bfloat16()
h2 = torch.empty_like(h)
for _ in range(3):
    if which == "l1":
        sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_GROUPED, out=h, activation="gelu", act_out=h2)
    elif which == "dh":
        sm.scatter2scatter(xg, w.view(E, de, d), order, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, out=h2,
                           activation="gelu", act_grad_of=h)
    elif which == "gather":
        sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_GROUPED, out=h)
    elif which == "gathers":  # gather, scattered output (S->S)
        sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_SCATTERED, out=h)
    elif which == "rowss":  # TMA rows, scattered output (G->S)
        sm.scatter2scatter(xg, w, order, 1, sm.GROUPED_TO_SCATTERED, out=h)
    elif which == "dhnone":
        sm.scatter2scatter(xg, w.view(E, de, d), order, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, out=h2)
    elif which == "dx":
        sm.scatter2scatter(h, w, order, 1, sm.GROUPED_TO_SCATTERED, transpose_w=True, out=xg)
    elif which == "rows":
        sm.scatter2scatter(xg, w, order, 1, sm.GROUPED_TO_GROUPED, out=h)
    elif which == "xtyboth":
        sm.group_xty(h, xg, order)
        sm.group_xty(xg, h, order)
    elif which == "xty":
        sm.group_xty(h, xg, order)
    elif which == "xtyal":  # bins that are multiples of 64 (no K tails)
        if _ == 0:
            ids_al = (torch.arange(n, device=dev) % E).view(T, k)
            r_al = sm.RoutingResult(ids_al, routing.p, routing.gate_full, renormalized=True, validate=False)
            order_al = sm.compute_grouped_order(r_al)
        sm.group_xty(h, xg, order_al)
    elif which == "cublas":  # dense library GEMM with the same FLOPs (n x d @ d x d_e)
        torch.matmul(xg, w[0])
    elif which == "xtysg":  # dW1 with X gathered by slot (no grouped copy)
        sm.kernels.group_xty_scattered(x, h, order, x_fan_out=k, y_grouped=True)
    elif which == "l1s":  # layer 1 on the routing-weight-scaled MLP path (bench's kernel)
        pf = routing.p.reshape(-1).float().contiguous()
        sm.kernels.scatter2scatter_scaled(x, w, order, k, sm.SCATTERED_TO_GROUPED, row_scale=pf, activation="gelu",
                                          out=h, act_out=h2)
    elif which == "dhs":  # dH with p scale + dp partials (bench's kernel)
        pf = routing.p.reshape(-1).float().contiguous()
        parts = torch.empty((n, sm.kernels.dp_parts(de)), dtype=torch.float32, device=dev)
        sm.kernels.scatter2scatter_scaled(xg, w.view(E, de, d), order, 1, sm.GROUPED_TO_GROUPED, row_scale=pf,
                                          activation="gelu", out=h2, act_grad_of=h, dp_partials=parts,
                                          transpose_w=True)
    elif which == "ofwd":  # scattered fan-out-1 input, scattered output, K = d_expert (C3 o-projection forward)
        sm.scatter2scatter(h, w.view(E, de, d), order, 1, sm.SCATTERED_TO_SCATTERED, out=xg)
    elif which == "l2":
        sm.scatter2scatter(h, w.view(E, de, d), order, 1, sm.GROUPED_TO_SCATTERED, out=xg)
torch.cuda.synchronize()
