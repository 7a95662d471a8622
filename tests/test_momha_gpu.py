"""Mixture-of-attention projections (moe_layers.py:406-482) vs the reference's outputs."""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from conftest import load_golden
from gpu_util import np_of, order_of, rel_err, routing_of, t

pytestmark = pytest.mark.gpu


def test_golden_momha_fp32():
    g = load_golden("momha")
    cfg = sm.MomhaConfig(d_model=16, d_head=4, num_heads=4, heads_per_expert=2, num_experts=3, k=2)
    wts = sm.MomhaWeights(wq=t(g["wq"]), wk=t(g["wk"]), wv=t(g["wv"]), wo=t(g["wo"]))
    routing = routing_of(g["idx"], g["p"], 3)
    order = order_of(g["idx"], 3)
    y, ctx = sm.momha_forward(t(g["x"]), wts, routing, order, cfg, int(g["seq_len"]))
    np.testing.assert_allclose(np_of(y), g["y"], rtol=1e-4, atol=1e-5)
    gr = sm.momha_backward(ctx, t(g["dy"]))
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dp"):
        got = getattr(gr, name)
        assert rel_err(got, g[name]) <= 1e-4, (name, rel_err(got, g[name]))


def test_momha_projection_shapes_c3_bf16():
    """C3 shape class (E=16, k=4, d_model=2048, d_proj=512): projections run and are finite."""
    cfg = sm.MomhaConfig(d_model=2048, d_head=128, num_heads=16, heads_per_expert=4, num_experts=16, k=4)
    seq, b = 512, 2
    x = (torch.rand((b * seq, 2048), device="cuda") * 2 - 1).to(torch.bfloat16)
    wts = sm.init_momha_weights(cfg, 0, dtype=torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(b * seq, 16, device="cuda"), 1), 4)
    order = sm.compute_grouped_order(routing)
    y, ctx = sm.momha_forward(x, wts, routing, order, cfg, seq)
    gr = sm.momha_backward(ctx, torch.ones_like(y))
    assert y.shape == (b * seq, 2048) and torch.isfinite(y.float()).all()
    assert torch.isfinite(gr.dwq.float()).all() and torch.isfinite(gr.dwo.float()).all()


def test_momha_bf16_matches_fp32_path():
    """bf16 MoMHA (tcgen05 projections + fused SDPA core) vs the fp32 path on the
    same bf16-rounded inputs: rel. err <= 2e-2 per output and gradient."""
    cfg = sm.MomhaConfig(d_model=256, d_head=64, num_heads=8, heads_per_expert=2, num_experts=8, k=4)
    seq, b = 256, 3
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.rand((b * seq, 256), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand((b * seq, 256), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    w16 = sm.init_momha_weights(cfg, 3, dtype=torch.bfloat16)
    w32 = sm.MomhaWeights(*(getattr(w16, f).float() for f in ("wq", "wk", "wv", "wo")))
    routing = sm.topk_select(torch.softmax(torch.randn(b * seq, 8, device="cuda", generator=g), 1), 4)
    order = sm.compute_grouped_order(routing)
    y16, c16 = sm.momha_forward(x, w16, routing, order, cfg, seq)
    y32, c32 = sm.momha_forward(x.float(), w32, routing, order, cfg, seq)
    assert rel_err(y16, y32.cpu().numpy()) <= 2e-2
    g16, g32 = sm.momha_backward(c16, dy), sm.momha_backward(c32, dy.float())
    for name in ("dx", "dwq", "dwk", "dwv", "dwo", "dp"):
        assert rel_err(getattr(g16, name), getattr(g32, name).cpu().numpy()) <= 2e-2, name


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_heads_to_grouped_matches_permute_and_group(dtype):
    """smoe_heads_to_grouped == (head layout -> slot rows) then group() by the order."""
    b, seq, k, h, dh, e = 3, 40, 4, 2, 64, 6
    g = torch.Generator(device="cuda").manual_seed(9)
    heads = torch.randn((b, h * k, seq, dh), device="cuda", generator=g).to(dtype)
    t = b * seq
    ids = torch.stack([torch.randperm(e, generator=torch.Generator().manual_seed(i))[:k] for i in range(t)]).cuda()
    routing = sm.RoutingResult(ids, torch.rand(t, k, device="cuda"), torch.zeros(t, e, device="cuda"),
                               renormalized=False, validate=False)
    order = sm.compute_grouped_order(routing)
    slots = heads.view(b, h, k, seq, dh).permute(0, 3, 2, 1, 4).reshape(t * k, h * dh)
    want = slots[order.o.long()]
    got = sm.kernels.heads_to_grouped(heads, order, k)
    assert torch.equal(got, want)


def test_momha_c3_full_size_vs_oracle():
    """C3 (E=16, k=4, d_model=2048, d_head=128, seq 4096, B=8 -> T=32768) in bf16 vs the oracle.

    dY is zero outside one sampled sequence b.  Attention never crosses a
    sequence, so every gradient then equals the oracle's gradients of that
    sequence alone (oracle/scattermlp_oracle.py momha_forward/backward,
    moe_layers.py:406-482): Y, dX and dp rows of sequence b, and the FULL weight
    gradients dWq, dWk, dWv, dWo — produced by the routed projection GEMMs at
    full C3 size (bins over all 32768 tokens, zero rows included).
    """
    from gpu_util import bf16_round
    from oracle import scattermlp_oracle as orc

    cfg = sm.MomhaConfig(d_model=2048, d_head=128, num_heads=16, heads_per_expert=4, num_experts=16, k=4)
    seq, b = 4096, 8
    rng = np.random.default_rng(7)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = (torch.rand((b * seq, 2048), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    wts = sm.init_momha_weights(cfg, 5, dtype=torch.bfloat16)
    logits = torch.randn((b * seq, 16), device="cuda", generator=g)
    routing = sm.topk_select(torch.softmax(logits, 1), 4)
    order = sm.compute_grouped_order(routing)
    sb = int(rng.integers(b))
    lo, hi = sb * seq, (sb + 1) * seq
    dy = torch.zeros((b * seq, 2048), device="cuda", dtype=torch.bfloat16)
    dy[lo:hi] = (torch.rand((seq, 2048), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    y, ctx = sm.momha_forward(x, wts, routing, order, cfg, seq)
    gr = sm.momha_backward(ctx, dy)
    torch.cuda.synchronize()

    xs = np_of(x[lo:hi])
    idx = routing.expert_idx[lo:hi].cpu().numpy()
    p = routing.p[lo:hi].cpu().numpy()
    wq, wk, wv, wo = (np_of(getattr(wts, f)) for f in ("wq", "wk", "wv", "wo"))
    want_y, st = orc.momha_forward(xs, wq, wk, wv, wo, idx, p, 16, seq, 128)
    want = orc.momha_backward(xs, wq, wk, wv, wo, p, st, np_of(dy[lo:hi]))
    assert rel_err(y[lo:hi], want_y) <= 2e-2
    errs = {"dx": rel_err(gr.dx[lo:hi], want[0]), "dp": rel_err(gr.dp[lo:hi], want[5]),
            "dwq": rel_err(gr.dwq, want[1]), "dwk": rel_err(gr.dwk, want[2]),
            "dwv": rel_err(gr.dwv, want[3]), "dwo": rel_err(gr.dwo, want[4])}
    assert all(v <= 2e-2 for v in errs.values()), errs
    # tokens outside the sampled sequence get no gradient
    assert float(gr.dx[:lo].abs().max() if lo else 0.0) == 0.0


def test_grouped_to_heads_inverts_heads_to_grouped():
    """grouped slot rows -> head layout -> grouped rows is the identity (bf16 and fp32)."""
    for dt in (torch.bfloat16, torch.float32):
        g = torch.Generator(device="cuda").manual_seed(3)
        b, seq, k, h, dh, e = 2, 96, 3, 2, 64, 6
        t = b * seq
        routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
        order = sm.compute_grouped_order(routing)
        rows = torch.randn(t * k, h * dh, device="cuda", generator=g).to(dt)
        heads = sm.kernels.grouped_to_heads(rows, order, k, b, seq, dh)
        # head layout (b, h*k, S, dh): head hh*k + j of token (b, s) = grouped row of slot (b*S+s)*k + j
        slots = rows[order.inverse().long()].view(b, seq, k, h, dh).permute(0, 3, 2, 1, 4).reshape(b, h * k, seq, dh)
        assert torch.equal(heads, slots)
        assert torch.equal(sm.kernels.heads_to_grouped(heads, order, k), rows)
        w = torch.rand(t * k, device="cuda", generator=g)
        acc = torch.float32 if dt == torch.bfloat16 else torch.float64   # the kernel's accumulate type
        want = (rows.to(acc) * w[order.o.long()].to(acc)[:, None]).to(dt)
        assert torch.equal(sm.kernels.scale_grouped_rows(rows, order, w), want)


def test_scatter2scatter_heads_matches_grouped_gemm_then_move():
    """The head-layout GEMM output (plain and the scaled act-grad + dp epilogue)
    equals the grouped-output GEMM followed by grouped_to_heads, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(11)
    b, seq, k, e, d_in, dh, hpe = 2, 192, 4, 8, 256, 128, 2
    d_out = dh * hpe
    t_ = b * seq
    routing = sm.topk_select(torch.softmax(torch.randn(t_, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    x = (torch.rand((t_, d_in), device="cuda", generator=g) * 2 - 1).bfloat16()
    w = ((torch.rand((e, d_in, d_out), device="cuda", generator=g) * 2 - 1) / 16).bfloat16()
    heads = sm.kernels.scatter2scatter_heads(x, w, order, k, False, batch=b, seq_len=seq, k=k, d_head=dh)
    ref = sm.kernels.grouped_to_heads(sm.scatter2scatter(x, w, order, k, sm.SCATTERED_TO_GROUPED), order, k, b, seq, dh)
    assert torch.equal(heads, ref)
    # transposed weights, grouped input, scaled identity act-grad with dp partials
    dyg = (torch.rand((t_ * k, d_out), device="cuda", generator=g) * 2 - 1).bfloat16()
    xg = (torch.rand((t_ * k, d_in), device="cuda", generator=g) * 2 - 1).bfloat16()
    wt = ((torch.rand((e, d_in, d_out), device="cuda", generator=g) * 2 - 1) / 16).bfloat16()
    p_flat = routing.p.reshape(-1).float().contiguous()
    parts_h = torch.empty((t_ * k, sm.kernels.dp_parts(d_in)), device="cuda")
    parts_g = torch.empty_like(parts_h)
    hx = sm.kernels.scatter2scatter_heads(dyg, wt, order, 1, True, batch=b, seq_len=seq, k=k, d_head=dh // 2,
                                          transpose_w=True, row_scale=p_flat, act_grad_of=xg, dp_partials=parts_h)
    gx = sm.kernels.scatter2scatter_scaled(dyg, wt, order, 1, sm.GROUPED_TO_GROUPED, row_scale=p_flat,
                                           activation="identity", out=torch.empty_like(xg), act_grad_of=xg,
                                           dp_partials=parts_g, transpose_w=True)
    assert torch.equal(hx, sm.kernels.grouped_to_heads(gx, order, k, b, seq, dh // 2))
    assert torch.equal(parts_h, parts_g)


@pytest.mark.parametrize("seed", range(10))
def test_momha_bf16_random_shapes_vs_oracle(seed):
    """Seeded random sweep of the bf16 MoMHA layer (head-layout q projection when
    d_head % 64 == 0, grouped slot rows otherwise; causal and not): batches of
    1-3 sequences of 1-96 tokens, k 1-4, d_head 8-128, against the oracle on the
    same bf16-rounded inputs (Y, dX, dp and all four weight gradients)."""
    from oracle import scattermlp_oracle as orc

    rng = np.random.default_rng(4000 + seed)
    k = int(rng.integers(1, 5))
    hpe = int(rng.choice([1, 2]))
    d_head = int(rng.choice([8, 32, 64, 128]))
    e = int(rng.integers(k, 17))
    d_model = int(8 * rng.integers(2, 33))
    b, seq = int(rng.integers(1, 4)), int(rng.choice([1, 17, 64, 96]))
    causal = bool(seed % 2 == 0)
    cfg = sm.MomhaConfig(d_model=d_model, d_head=d_head, num_heads=k * hpe, heads_per_expert=hpe,
                         num_experts=e, k=k, causal=causal)
    wts = sm.init_momha_weights(cfg, seed, dtype=torch.bfloat16)
    n = b * seq
    x = t(rng.uniform(-1, 1, (n, d_model)).astype(np.float32), torch.bfloat16)
    dy = t(rng.uniform(-1, 1, (n, d_model)).astype(np.float32), torch.bfloat16)
    idx = np.stack([rng.permutation(e)[:k] for _ in range(n)])
    p = rng.uniform(0.05, 1.0, (n, k)).astype(np.float32)
    p /= p.sum(1, keepdims=True)
    routing, order = routing_of(idx, p, e), order_of(idx, e)
    y, ctx = sm.momha_forward(x, wts, routing, order, cfg, seq)
    gr = sm.momha_backward(ctx, dy)
    wq, wk, wv, wo = (np_of(getattr(wts, f)) for f in ("wq", "wk", "wv", "wo"))
    want_y, st = orc.momha_forward(np_of(x), wq, wk, wv, wo, idx, p, e, seq, d_head, causal)
    want = orc.momha_backward(np_of(x), wq, wk, wv, wo, p, st, np_of(dy))
    case = (b, seq, k, hpe, d_head, e, d_model, causal)
    assert rel_err(y, want_y) <= 2e-2, case
    for j, name in enumerate(("dx", "dwq", "dwk", "dwv", "dwo")):
        assert rel_err(getattr(gr, name), want[j]) <= 2e-2, (name, rel_err(getattr(gr, name), want[j]), case)
    absdot = (np.abs(np_of(dy)).astype(np.float64)[:, None, :] * np.abs(st["y_hat"]).reshape(n, k, d_model)).sum(-1)
    err = np.abs(np_of(gr.dp).astype(np.float64) - want[5])
    assert np.all(err <= 2e-2 * absdot + 1e-6), ("dp", case)
