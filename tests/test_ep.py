"""Expert-parallel SMoE MLP (paper_2403_08245_b200.ep).

* CPU, world_size 2 (and 4), gloo backend: the count exchange, all-to-all-v
  dispatch / return, local grouped order and source-side un-permute + combine
  reproduce the single-process oracle on the concatenated batch (the EP path
  runs the routing-weight-scaled MLP form: equal to the literal form up to
  float32 rounding).
* GPU (1 B200, NCCL world 1): the EP path through the CUDA ops is
  bit-identical to the single-GPU smoe_mlp_forward / backward.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scattermlp_oracle as orc

T_LOCAL, D, DE, E, K = 24, 16, 32, 8, 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(world):
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (world * T_LOCAL, D)).astype(np.float32)
    w1 = (rng.uniform(-1, 1, (E, D, DE)) / np.sqrt(D)).astype(np.float32)
    w2 = (rng.uniform(-1, 1, (E, DE, D)) / np.sqrt(DE)).astype(np.float32)
    idx = np.stack([rng.permutation(E)[:K] for _ in range(world * T_LOCAL)]).astype(np.int64)
    idx[:5] = np.arange(K)              # skewed rows
    p = rng.random((world * T_LOCAL, K)).astype(np.float32) + 0.1
    p /= p.sum(1, keepdims=True)
    dy = rng.uniform(-1, 1, (world * T_LOCAL, D)).astype(np.float32)
    return x, w1, w2, idx, p, dy


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from ep_cpu_ops import CpuOps
        import paper_2403_08245_b200 as sm
        from paper_2403_08245_b200.ep import ExpertParallelSmoeMlp

        x, w1, w2, idx, p, dy = _problem(world)
        sl = slice(rank * T_LOCAL, (rank + 1) * T_LOCAL)
        el = E // world
        ep = ExpertParallelSmoeMlp(torch.from_numpy(w1[rank * el:(rank + 1) * el]),
                                   torch.from_numpy(w2[rank * el:(rank + 1) * el]), E, ops=CpuOps())
        routing = sm.RoutingResult(torch.from_numpy(idx[sl]), torch.from_numpy(p[sl]), torch.zeros(T_LOCAL, E),
                                   renormalized=False, validate=False)
        y, ctx = ep.forward(torch.from_numpy(x[sl]), routing)
        g = ep.backward(ctx, torch.from_numpy(dy[sl]))
        q.put((rank, y.numpy(), g.dx.numpy(), g.dp.numpy(), g.dw1.numpy(), g.dw2.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_gloo_matches_single_process_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = {}
    for _ in range(world):
        r = q.get(timeout=120)
        results[r[0]] = r[1:]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x, w1, w2, idx, p, dy = _problem(world)
    y_ref, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, E)
    dx_ref, dw1_ref, dw2_ref, dp_ref = orc.smoe_mlp_backward(x, w1, w2, p, st, dy)
    el = E // world
    for rank in range(world):
        y, dx, dp, dw1, dw2 = results[rank]
        sl = slice(rank * T_LOCAL, (rank + 1) * T_LOCAL)
        np.testing.assert_allclose(y, y_ref[sl], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(dx, dx_ref[sl], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(dp, dp_ref[sl], rtol=1e-5, atol=1e-6)
        # expert weight gradients stay local: this rank's slice of the global dW
        np.testing.assert_allclose(dw1, dw1_ref[rank * el:(rank + 1) * el], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(dw2, dw2_ref[rank * el:(rank + 1) * el], rtol=1e-5, atol=1e-6)


def test_local_order_from_counts():
    from paper_2403_08245_b200.ep import local_order_from_counts
    counts = torch.tensor([[2, 0, 1], [1, 3, 0]])       # 2 sources x 3 local experts
    o, off = local_order_from_counts(counts)
    # recv layout: src0 = [e0 e0 e2], src1 = [e0 e1 e1 e1]; rows 0..6
    assert off.tolist() == [0, 3, 6, 7]
    assert o.tolist() == [0, 1, 3, 4, 5, 6, 2]


@pytest.mark.gpu
def test_ep_world1_nccl_bit_identical_to_single_gpu():
    import paper_2403_08245_b200 as sm
    from paper_2403_08245_b200.ep import ExpertParallelSmoeMlp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        t, d, de, e, k = 2048, 256, 512, 8, 2
        g = torch.Generator(device="cuda").manual_seed(0)
        x = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        dy = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        w1 = ((torch.rand(e, d, de, device="cuda", generator=g) * 2 - 1) / 16).bfloat16()
        w2 = ((torch.rand(e, de, d, device="cuda", generator=g) * 2 - 1) / 22).bfloat16()
        routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
        order = sm.compute_grouped_order(routing)
        prev = sm.moe_layers.set_scaled(True)    # the NCCL EP path runs the routing-weight-scaled form
        try:
            y_ref, c = sm.smoe_mlp_forward(x, w1, w2, routing, order)
            gr = sm.smoe_mlp_backward(c, dy)
        finally:
            sm.moe_layers.set_scaled(prev)
        ep = ExpertParallelSmoeMlp(w1, w2, e)
        y, ctx = ep.forward(x, routing)
        ge = ep.backward(ctx, dy)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
        assert torch.equal(ge.dx, gr.dx)
        assert torch.equal(ge.dp, gr.dp)
        assert torch.equal(ge.dw1, gr.dw1)
        assert torch.equal(ge.dw2, gr.dw2)
    finally:
        dist.destroy_process_group()
