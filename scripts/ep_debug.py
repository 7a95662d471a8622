"""Debug: 2 processes sharing the GPU, scaled peer EP; where does dW2 differ?"""
import os
import socket
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2403_08245_b200 as sm
    from paper_2403_08245_b200 import kernels as K
    from paper_2403_08245_b200.ep_peer import PeerExpertParallelSmoeMlp
    from test_ep_peer import _problem, SHAPES
    torch.cuda.set_device(0)
    E, KK, T = SHAPES["c1"][:3]
    x, dy, w1, w2, logits = _problem(world, "c1")
    routing = sm.topk_select(torch.softmax(logits, 1), KK)
    order = sm.compute_grouped_order(routing)
    sm.moe_layers.set_scaled(True)
    y_ref, c = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    g_ref = sm.smoe_mlp_backward(c, dy)
    sl = slice(rank * T, (rank + 1) * T)
    el = E // world
    es = slice(rank * el, (rank + 1) * el)
    ep = PeerExpertParallelSmoeMlp(w1[es].contiguous(), w2[es].contiguous(), E, KK, max_tokens=T, timeout_s=60.0,
                                   scaled=True)
    rt = sm.RoutingResult(routing.expert_idx[sl].contiguous(), routing.p[sl].contiguous(),
                          routing.gate_full[sl].contiguous(), renormalized=True, validate=False)
    for it in range(3):
        y, ctx = ep.forward(x[sl].contiguous(), rt)
        hsave = ctx.h.clone()
        gr = ep.backward(ctx, dy[sl].contiguous())
        torch.cuda.synchronize()
        dist.barrier()
        dyl = ep.recv_dy.view(torch.bfloat16, (ep.cap, ep.d))
        redo = K.group_xty(hsave, dyl, ctx.order_loc)
        per_e = [bool(torch.equal(gr.dw2[i], g_ref.dw2[es][i])) for i in range(el)]
        # layer 1 recomputed (ungated) on the resident received rows
        n_recv = int(ctx.order_loc.bin_offsets[-1])
        h_pre2 = torch.empty_like(ep.h_pre)
        h2 = torch.empty_like(ep.h)
        K.scatter2scatter_scaled(ep.recv_x.view(torch.bfloat16, (ep.cap, ep.d)), ep.w1, ctx.order_loc, 1,
                                 sm.GROUPED_TO_GROUPED, row_scale=ep._recv_p(), activation="gelu", out=h_pre2,
                                 act_out=h2)
        torch.cuda.synchronize()
        bad = (h2[:n_recv] != hsave[:n_recv]).any(1).nonzero().flatten()
        src = ep.recv_src.view(torch.int32, (ep.cap,))[:n_recv]
        if bad.numel():
            print(rank, it, "h rows differ:", bad.numel(), "of", n_recv, "first", bad[:8].tolist(), "srcs",
                  torch.bincount(src[bad].long(), minlength=2).tolist(), "pre differs",
                  int((h_pre2[:n_recv] != ep.h_pre[:n_recv]).any(1).sum()), flush=True)
        print(rank, it, "dw2 eq", per_e, "redo==ref", torch.equal(redo, g_ref.dw2[es]), "redo==ep",
              torch.equal(redo, gr.dw2), "y", torch.equal(y, y_ref[sl]), "err", int(ep.err.item()), flush=True)
    ep.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port), nprocs=2)
