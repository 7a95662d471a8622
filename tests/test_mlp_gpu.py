"""SMoE MLP fwd+bwd parity (moe_layers.py:140-211) on the GPU.

* golden cases (reference outputs, fp32 check mode): elementwise rtol 1e-5 and
  relative Frobenius <= 1e-4;
* C0 full size (T=4096, d=512, d_e=1024, E=8, k=2) vs the oracle in fp32
  (<= 1e-4) and in bf16 with bf16-rounded oracle inputs (<= 2e-2);
* C1 / C2 full sizes in bf16: sampled tokens checked exactly against the
  per-token oracle (Y, dX, dp are token-local), and dW1 / dW2 column slices of
  the longest expert bins recomputed in f64 over the whole bin.
"""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from conftest import load_golden
from gpu_util import bf16_round, np_of, order_of, rel_err, routing_of, t
from oracle import scattermlp_oracle as orc

pytestmark = pytest.mark.gpu


def _run(x, w1, w2, idx, p, e, act, dtype, engine=None):
    if engine:
        sm.set_engine(engine)
    try:
        routing = routing_of(idx, p, e)
        order = order_of(idx, e)
        y, ctx = sm.smoe_mlp_forward(t(x, dtype), t(w1, dtype), t(w2, dtype), routing, order, activation=act)
        return y, ctx
    finally:
        sm.set_engine("auto")


def test_golden_mlp_fp32():
    g = load_golden("mlp")
    for j in range(int(g["num_mlp"])):
        pre = f"mlp{j}_"
        act = str(g[pre + "act"])
        y, ctx = _run(g[pre + "x"], g[pre + "w1"], g[pre + "w2"], g[pre + "idx"], g[pre + "p"],
                      int(g[pre + "E"]), act, torch.float32)
        np.testing.assert_allclose(np_of(y), g[pre + "y"], rtol=1e-5, atol=1e-6, err_msg=f"{j}")
        np.testing.assert_allclose(np_of(y), g[pre + "y_naive"], rtol=1e-5, atol=1e-6)
        gr = sm.smoe_mlp_backward(ctx, t(g[pre + "dy"]))
        for got, name in ((gr.dx, "dx"), (gr.dw1, "dw1"), (gr.dw2, "dw2"), (gr.dp, "dp")):
            np.testing.assert_allclose(np_of(got), g[pre + name], rtol=1e-5, atol=1e-5, err_msg=f"{j}:{name}")
            assert rel_err(got, g[pre + name]) <= 1e-4, (j, name)


def test_golden_mlp_bf16():
    g = load_golden("mlp")
    for j in range(int(g["num_mlp"])):
        pre = f"mlp{j}_"
        act = str(g[pre + "act"])
        x, w1, w2 = (bf16_round(g[pre + n]) for n in ("x", "w1", "w2"))
        dy = bf16_round(g[pre + "dy"])
        want_y, st = orc.smoe_mlp_forward(x, w1, w2, g[pre + "idx"], g[pre + "p"], int(g[pre + "E"]), act)
        want = orc.smoe_mlp_backward(x, w1, w2, g[pre + "p"], st, dy, act)
        y, ctx = _run(x, w1, w2, g[pre + "idx"], g[pre + "p"], int(g[pre + "E"]), act, torch.bfloat16)
        assert rel_err(y, want_y) <= 2e-2
        gr = sm.smoe_mlp_backward(ctx, t(dy, torch.bfloat16))
        for got, w_, name in zip((gr.dx, gr.dw1, gr.dw2, gr.dp), want, ("dx", "dw1", "dw2", "dp")):
            assert rel_err(got, w_) <= 2e-2, (j, name, rel_err(got, w_))


def _c0(dtype_np_round):
    x, w1, w2, idx, p, dy = orc.mlp_problem(4096, 512, 1024, 8, 2, seed=0)
    if dtype_np_round:
        x, w1, w2, dy = (bf16_round(a) for a in (x, w1, w2, dy))
    return x, w1, w2, idx, p, dy


def test_c0_fp32_check_mode():
    x, w1, w2, idx, p, dy = _c0(False)
    want_y, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, 8)
    want = orc.smoe_mlp_backward(x, w1, w2, p, st, dy)
    y, ctx = _run(x, w1, w2, idx, p, 8, "gelu", torch.float32)
    assert rel_err(y, want_y) <= 1e-4
    gr = sm.smoe_mlp_backward(ctx, t(dy))
    for got, w_, name in zip((gr.dx, gr.dw1, gr.dw2, gr.dp), want, ("dx", "dw1", "dw2", "dp")):
        assert rel_err(got, w_) <= 1e-4, (name, rel_err(got, w_))


@pytest.mark.parametrize("engine,scaled", [("simt", True), ("auto", True), ("auto", False)])
def test_c0_bf16(engine, scaled):
    """scaled: the routing weight moved through layer 2 (dp from the dH epilogue);
    False: the reference's literal sequence (combine, dp from the retained output)."""
    x, w1, w2, idx, p, dy = _c0(True)
    want_y, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, 8)
    want = orc.smoe_mlp_backward(x, w1, w2, p, st, dy)
    sm.set_engine(engine)
    prev = sm.moe_layers.set_scaled(scaled)
    try:
        y, ctx = _run(x, w1, w2, idx, p, 8, "gelu", torch.bfloat16)
        if engine == "auto":
            assert (ctx.scaled is not None) == scaled
        gr = sm.smoe_mlp_backward(ctx, t(dy, torch.bfloat16))
    finally:
        sm.set_engine("auto")
        sm.moe_layers.set_scaled(prev)
    assert rel_err(y, want_y) <= 2e-2
    for got, w_, name in zip((gr.dx, gr.dw1, gr.dw2, gr.dp), want, ("dx", "dw1", "dw2", "dp")):
        assert rel_err(got, w_) <= 2e-2, (name, rel_err(got, w_))


def _sampled_large(tokens, d, de, e, k, n_sample=48, seed=0):
    """Full-size bf16 fwd+bwd; sampled tokens vs the per-token oracle."""
    rng = np.random.default_rng(seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / np.sqrt(d)).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / np.sqrt(de)).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    wg = (torch.rand((d, e), generator=g, device="cuda") * 2 - 1) / np.sqrt(d)
    routing = sm.topk_select(sm.gate_forward(x.float(), wg), k)
    order = sm.compute_grouped_order(routing)
    y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    gr = sm.smoe_mlp_backward(ctx, dy)
    torch.cuda.synchronize()
    toks = np.sort(rng.choice(tokens, n_sample, replace=False))
    idx = routing.expert_idx.cpu().numpy()
    p = routing.p.cpu().numpy()
    xs = np_of(x[toks]); dys = np_of(dy[toks])
    w1n = {}; w2n = {}
    want_y = np.zeros((n_sample, d)); want_dx = np.zeros((n_sample, d)); want_dp = np.zeros((n_sample, k))
    for r, tok in enumerate(toks):
        for j in range(k):
            ee = int(idx[tok, j])
            if ee not in w1n:
                w1n[ee] = np_of(w1[ee]).astype(np.float64)
                w2n[ee] = np_of(w2[ee]).astype(np.float64)
            hp = xs[r].astype(np.float64) @ w1n[ee]
            h = orc.act(hp, "gelu")
            yh = h @ w2n[ee]
            want_y[r] += p[tok, j] * yh
            want_dp[r, j] = dys[r].astype(np.float64) @ yh
            dh = (p[tok, j] * dys[r].astype(np.float64)) @ w2n[ee].T * orc.act_grad(hp, "gelu")
            want_dx[r] += dh @ w1n[ee].T
    assert rel_err(y[toks], want_y) <= 2e-2
    assert rel_err(gr.dx[toks], want_dx) <= 2e-2
    assert rel_err(gr.dp[toks], want_dp) <= 2e-2
    _dw_slices(x, w1, w2, dy, routing, order, gr, k, n_experts=4 if e <= 8 else 8, rng=rng)
    return y, gr


def _dw_slices(x, w1, w2, dy, routing, order, gr, k, n_experts, rng, n_cols=16, act="gelu"):
    """Weight gradients checked exactly over whole expert bins.

    For n_experts experts and n_cols sampled columns each, the f64 oracle
    (oracle/scattermlp_oracle.py's MLP restated per bin, kernels.py:329-361)
    recomputes over the expert's FULL bin:
      dW2[e][:, c] = act(X_bin W1[e])^T (p * dY)_bin[:, c]           (all d_expert rows)
      dW1[e][:, c] = X_bin^T ((p * dY)_bin W2[e][c, :]^T * act'(X_bin W1[e][:, c]))
    i.e. the grouped-K GEMMs at the bin lengths they run at in the benchmark
    (about 8192 rows at C1, 4096 at C2), not a small-shape stand-in.
    """
    off = order.bin_offsets.cpu().numpy().astype(np.int64)
    o = order.o.cpu().numpy().astype(np.int64)
    p_flat = routing.p.reshape(-1).float().cpu().numpy().astype(np.float64)
    counts = np.diff(off)
    experts = np.argsort(-counts, kind="stable")[:n_experts]       # the longest bins (the K the bench runs)
    xn = np_of(x).astype(np.float64)
    dyn = np_of(dy).astype(np.float64)
    d, de = w1.shape[1], w1.shape[2]
    for e in experts:
        e = int(e)
        slots = o[off[e]:off[e + 1]]
        toks = slots // k
        xb = xn[toks]
        dyb = p_flat[slots][:, None] * dyn[toks]
        w1e = np_of(w1[e]).astype(np.float64)
        w2e = np_of(w2[e]).astype(np.float64)
        c2 = np.sort(rng.choice(d, n_cols, replace=False))
        c1 = np.sort(rng.choice(de, n_cols, replace=False))
        hpre = xb @ w1e                                         # [bin, d_expert]
        want_dw2 = orc.act(hpre, act).T @ dyb[:, c2]            # [d_expert, n_cols]
        dh = (dyb @ w2e[c1, :].T) * orc.act_grad(hpre[:, c1], act)
        want_dw1 = xb.T @ dh                                    # [d_model, n_cols]
        err2 = rel_err(gr.dw2[e][:, c2], want_dw2)
        err1 = rel_err(gr.dw1[e][:, c1], want_dw1)
        assert err2 <= 2e-2 and err1 <= 2e-2, (e, int(counts[e]), err1, err2)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_full_size_sampled(cfg):
    if cfg == "C1":
        _sampled_large(32768, 4096, 14336, 8, 2)
    else:
        _sampled_large(32768, 4096, 1792, 64, 8)


def test_smoe_mlp_module_autograd():
    g = load_golden("mlp")
    pre = "mlp0_"
    cfg = sm.SmoeMlpConfig(d_model=32, d_expert=48, num_experts=4, k=2)
    mod = sm.SmoeMlp(cfg, dtype=torch.float32)
    with torch.no_grad():
        mod.w1.copy_(t(g[pre + "w1"]))
        mod.w2.copy_(t(g[pre + "w2"]))
    routing = routing_of(g[pre + "idx"], g[pre + "p"], 4)
    order = order_of(g[pre + "idx"], 4)
    x = t(g[pre + "x"]).requires_grad_(True)
    y = mod(x, routing, order)
    y.backward(t(g[pre + "dy"]))
    np.testing.assert_allclose(np_of(y), g[pre + "y"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np_of(x.grad), g[pre + "dx"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(np_of(mod.w1.grad), g[pre + "dw1"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(np_of(mod.w2.grad), g[pre + "dw2"], rtol=1e-5, atol=1e-5)


def test_train_equals_infer_and_relabel_invariance():
    """test_moe_layers.py:111-138 on the GPU (fp32)."""
    g = load_golden("mlp")
    pre = "mlp0_"
    y, _ = _run(g[pre + "x"], g[pre + "w1"], g[pre + "w2"], g[pre + "idx"], g[pre + "p"], 4, "gelu", torch.float32)
    routing = routing_of(g[pre + "idx"], g[pre + "p"], 4)
    order = order_of(g[pre + "idx"], 4)
    y_inf, _ = sm.smoe_mlp_forward(t(g[pre + "x"]), t(g[pre + "w1"]), t(g[pre + "w2"]), routing, order,
                                   training=False)
    np.testing.assert_allclose(np_of(y_inf), np_of(y), rtol=1e-5, atol=1e-6)
    perm = np.array([2, 0, 3, 1])
    inv = np.argsort(perm)
    y2, _ = _run(g[pre + "x"], g[pre + "w1"][inv], g[pre + "w2"][inv], perm[g[pre + "idx"]], g[pre + "p"], 4,
                 "gelu", torch.float32)
    np.testing.assert_allclose(np_of(y2), np_of(y), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("act", ["gelu", "silu", "relu"])
@pytest.mark.parametrize("flavor", ["gate", "skewed"])
def test_scaled_path_matches_literal_path(act, flavor):
    """The routing-weight-scaled MLP (p through layer 2, dp from the dH epilogue)
    against the literal sequence, bf16, ragged bins and partial tiles."""
    g = torch.Generator(device="cuda").manual_seed(3)
    tokens, d, de, e, k = 1000, 136, 264, 6, 2
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    logits = torch.randn(tokens, e, device="cuda", generator=g)
    if flavor == "skewed":
        logits[:, 0] += 6.0
    routing = sm.topk_select(torch.softmax(logits, 1), k)
    order = sm.compute_grouped_order(routing)
    out = {}
    for scaled in (True, False):
        prev = sm.moe_layers.set_scaled(scaled)
        try:
            y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order, activation=act)
            assert (ctx.scaled is not None) == scaled
            gr = sm.smoe_mlp_backward(ctx, dy)
        finally:
            sm.moe_layers.set_scaled(prev)
        out[scaled] = (y, gr.dx, gr.dw1, gr.dw2, gr.dp)
    for name, a, b in zip(("y", "dx", "dw1", "dw2", "dp"), out[True], out[False]):
        assert rel_err(a, np_of(b)) <= 1e-2, (name, rel_err(a, np_of(b)))


@pytest.mark.parametrize("tokens,d,de,e,k,flavor", [
    (1, 64, 128, 1, 1, "gate"),          # one token, one expert
    (3, 64, 64, 4, 2, "gate"),           # fewer rows than one tile
    (513, 128, 192, 16, 4, "all_to_one"),  # every token to experts 0..3, 12 empty bins
    (2048, 256, 256, 128, 8, "gate"),    # 128 experts (largest on the CTA-pair engine)
])
def test_scaled_mlp_edge_cases_vs_oracle(tokens, d, de, e, k, flavor):
    rng = np.random.default_rng(tokens + e)
    x = bf16_round(rng.uniform(-1, 1, (tokens, d)).astype(np.float32))
    w1 = bf16_round((rng.uniform(-1, 1, (e, d, de)) / np.sqrt(d)).astype(np.float32))
    w2 = bf16_round((rng.uniform(-1, 1, (e, de, d)) / np.sqrt(de)).astype(np.float32))
    dy = bf16_round(rng.uniform(-1, 1, (tokens, d)).astype(np.float32))
    if flavor == "all_to_one":
        idx = np.tile(np.arange(k), (tokens, 1))
    else:
        idx = np.stack([rng.permutation(e)[:k] for _ in range(tokens)])
    p = rng.uniform(0.05, 1.0, (tokens, k)).astype(np.float32)
    p /= p.sum(1, keepdims=True)
    want_y, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, e)
    want = orc.smoe_mlp_backward(x, w1, w2, p, st, dy)
    y, ctx = _run(x, w1, w2, idx, p, e, "gelu", torch.bfloat16)
    assert ctx.scaled is not None
    gr = sm.smoe_mlp_backward(ctx, t(dy, torch.bfloat16))
    assert rel_err(y, want_y) <= 2e-2
    for got, w_, name in zip((gr.dx, gr.dw1, gr.dw2), want[:3], ("dx", "dw1", "dw2")):
        assert rel_err(got, w_) <= 2e-2, (name, rel_err(got, w_))
    # dp entries are single dot products: with few tokens the Frobenius norm is
    # dominated by cancelling ones, so bound each by its absolute dot product
    absdot = np.abs(dy).astype(np.float64)[:, None, :] * np.abs(st["y_hat"]).reshape(tokens, k, d)
    absdot = absdot.sum(-1)
    err = np.abs(np_of(gr.dp).astype(np.float64) - want[3])
    assert np.all(err <= 2e-2 * absdot + 1e-6), float((err / np.maximum(absdot, 1e-30)).max())
    if tokens >= 64:
        assert rel_err(gr.dp, want[3]) <= 2e-2


def test_training_step_cuda_graph_capture_bit_identical():
    """The whole step (routing sort, forward, backward) captures into one CUDA
    graph (no host syncs, no allocations inside the library) and replays
    bit-identically to eager execution."""
    g = torch.Generator(device="cuda").manual_seed(9)
    tokens, d, de, e, k = 2048, 256, 512, 8, 2
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).to(torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)

    def step():
        order = sm.compute_grouped_order(routing)
        y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
        return y, sm.smoe_mlp_backward(ctx, dy)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y_g, gr_g = step()
    y_e, gr_e = step()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_g, y_e)
    for a, b in ((gr_g.dx, gr_e.dx), (gr_g.dw1, gr_e.dw1), (gr_g.dw2, gr_e.dw2), (gr_g.dp, gr_e.dp)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("training", [True, False])
def test_zero_tokens(training):
    """A batch with no tokens (an EP rank that receives nothing): empty outputs, zero dW."""
    e, d, de, k = 4, 64, 128, 2
    w1 = torch.zeros((e, d, de), dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros((e, de, d), dtype=torch.bfloat16, device="cuda")
    x = torch.zeros((0, d), dtype=torch.bfloat16, device="cuda")
    routing = sm.RoutingResult(expert_idx=torch.zeros((0, k), dtype=torch.int64, device="cuda"),
                               p=torch.zeros((0, k), dtype=torch.float32, device="cuda"),
                               gate_full=torch.zeros((0, e), device="cuda"), renormalized=False, validate=False)
    order = sm.compute_grouped_order(routing, e)
    y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order, training=training)
    assert tuple(y.shape) == (0, d)
    if training:
        gr = sm.smoe_mlp_backward(ctx, torch.zeros((0, d), dtype=torch.bfloat16, device="cuda"))
        torch.cuda.synchronize()
        assert tuple(gr.dx.shape) == (0, d) and tuple(gr.dp.shape) == (0, k)
        assert float(gr.dw1.abs().max()) == 0.0 and float(gr.dw2.abs().max()) == 0.0


def test_on_dx_hook_fires_before_dw1_with_final_dx():
    """smoe_mlp_backward(on_dx=...) hands over dX and dp as soon as their kernels
    are enqueued; the tensors are the returned gradients (bit-identical values)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    tokens, d, de, e, k = 1024, 256, 512, 8, 2
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).to(torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    seen = []
    y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    gr = sm.smoe_mlp_backward(ctx, dy, on_dx=lambda dx, dp: seen.append((dx.clone(), dp.clone())))
    assert len(seen) == 1
    torch.cuda.synchronize()
    assert torch.equal(seen[0][0], gr.dx) and torch.equal(seen[0][1], gr.dp)
    y2, ctx2 = sm.smoe_mlp_forward(x, w1, w2, routing, order)
    gr2 = sm.smoe_mlp_backward(ctx2, dy)
    for a, b in ((gr.dx, gr2.dx), (gr.dw1, gr2.dw1), (gr.dw2, gr2.dw2), (gr.dp, gr2.dp)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("tokens,e", [(1000, 6), (3, 4)])
def test_grouped_layer1_forward_bit_identical(tokens, e):
    """SMOE_L1_GROUPED: layer 1 fed by a grouped copy of X (TMA) instead of the
    in-GEMM row gather — same K order per output element, so bit-identical."""
    g = torch.Generator(device="cuda").manual_seed(11)
    d, de, k = 136, 264, 2
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).to(torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    out = {}
    prev = sm.moe_layers._L1_GROUPED
    try:
        for grouped in (False, True):
            sm.moe_layers._L1_GROUPED = grouped
            y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order)
            assert ctx.scaled is not None
            gr = sm.smoe_mlp_backward(ctx, dy)
            out[grouped] = (y, ctx.h_pre, gr.dx, gr.dw1, gr.dw2, gr.dp)
    finally:
        sm.moe_layers._L1_GROUPED = prev
    for name, a, b in zip(("y", "h_pre", "dx", "dw1", "dw2", "dp"), out[False], out[True]):
        assert torch.equal(a, b), name


@pytest.mark.parametrize("seed", range(12))
def test_scaled_mlp_random_shapes_vs_oracle(seed):
    """Seeded random sweep of the bf16 training path (routing-weight-scaled form,
    dp from the dH epilogue): expert counts 1..128, fan-out 1..8, widths from 8,
    one-token batches, all three activations — Y, dX, dW1, dW2, dp vs the oracle."""
    rng = np.random.default_rng(2000 + seed)
    e = int(rng.choice([1, 2, 5, 8, 16, 40, 128]))
    k = int(rng.integers(1, min(e, 8) + 1))
    tokens = int(rng.choice([1, 3, 64, 257, 900]))
    d = 8 if seed == 4 else int(8 * rng.integers(1, 40))
    de = 8 if seed == 7 else int(8 * rng.integers(1, 60))
    act = ["gelu", "silu", "relu"][seed % 3]
    x = bf16_round(rng.uniform(-1, 1, (tokens, d)).astype(np.float32))
    w1 = bf16_round((rng.uniform(-1, 1, (e, d, de)) / np.sqrt(d)).astype(np.float32))
    w2 = bf16_round((rng.uniform(-1, 1, (e, de, d)) / np.sqrt(de)).astype(np.float32))
    dy = bf16_round(rng.uniform(-1, 1, (tokens, d)).astype(np.float32))
    idx = np.stack([rng.permutation(e)[:k] for _ in range(tokens)])
    p = rng.uniform(0.05, 1.0, (tokens, k)).astype(np.float32)
    p /= p.sum(1, keepdims=True)
    want_y, st = orc.smoe_mlp_forward(x, w1, w2, idx, p, e, activation=act)
    want = orc.smoe_mlp_backward(x, w1, w2, p, st, dy, activation=act)
    y, ctx = _run(x, w1, w2, idx, p, e, act, torch.bfloat16)
    assert ctx.scaled is not None
    gr = sm.smoe_mlp_backward(ctx, t(dy, torch.bfloat16))
    case = (tokens, d, de, e, k, act)
    assert rel_err(y, want_y) <= 2e-2, case
    for got, w_, name in zip((gr.dx, gr.dw1, gr.dw2), want[:3], ("dx", "dw1", "dw2")):
        assert rel_err(got, w_) <= 2e-2, (name, rel_err(got, w_), case)
    # dp: each entry one dot product, bounded by its absolute dot product
    absdot = (np.abs(dy).astype(np.float64)[:, None, :] * np.abs(st["y_hat"]).reshape(tokens, k, d)).sum(-1)
    err = np.abs(np_of(gr.dp).astype(np.float64) - want[3])
    assert np.all(err <= 2e-2 * absdot + 1e-6), (float((err / np.maximum(absdot, 1e-30)).max()), case)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_full_size_token_permutation_equivariance(cfg):
    """A size-independent property at the full BASELINE shapes: permuting the
    tokens (and their routing) permutes Y, dX and dp BIT-EXACTLY — each output
    row is computed from its own slot rows in a fixed K order whatever its place
    in the expert bins — while dW1 / dW2 (sums over the bins, whose row order
    changes) agree to fp32 summation-order rounding."""
    tokens, d, de, e, k = (32768, 4096, 14336, 8, 2) if cfg == "C1" else (32768, 4096, 1792, 64, 8)
    g = torch.Generator(device="cuda").manual_seed(17)
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / np.sqrt(d)).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / np.sqrt(de)).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)
    perm = torch.randperm(tokens, generator=g, device="cuda")

    def run(xx, dyy, ids, p):
        rt = sm.RoutingResult(ids, p, torch.zeros((tokens, e), device="cuda"), renormalized=True, validate=False)
        order = sm.compute_grouped_order(rt)
        y, ctx = sm.smoe_mlp_forward(xx, w1, w2, rt, order)
        return y, sm.smoe_mlp_backward(ctx, dyy)

    y0, g0 = run(x, dy, routing.expert_idx, routing.p)
    y1, g1 = run(x[perm].contiguous(), dy[perm].contiguous(), routing.expert_idx[perm].contiguous(),
                 routing.p[perm].contiguous())
    assert torch.equal(y1, y0[perm])
    assert torch.equal(g1.dx, g0.dx[perm])
    assert torch.equal(g1.dp, g0.dp[perm])
    assert rel_err(g1.dw1, np_of(g0.dw1)) <= 2e-3
    assert rel_err(g1.dw2, np_of(g0.dw2)) <= 2e-3


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_full_size_expert_relabel_invariance(cfg):
    """Relabelling the experts (ids through a permutation sigma, weight stacks
    permuted to match) moves each expert's bin to another place in the grouped
    order but keeps its rows and their order: Y, dX, dp and every expert's
    dW1 / dW2 are bit-identical at the full BASELINE shapes (bin offsets,
    tile-to-expert mapping and per-expert schedules exercised at size)."""
    tokens, d, de, e, k = (32768, 4096, 14336, 8, 2) if cfg == "C1" else (32768, 4096, 1792, 64, 8)
    g = torch.Generator(device="cuda").manual_seed(23)
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / np.sqrt(d)).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / np.sqrt(de)).to(torch.bfloat16)
    dy = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    logits = torch.randn(tokens, e, device="cuda", generator=g)
    logits[:, 0] += 1.0                                   # uneven bins
    routing = sm.topk_select(torch.softmax(logits, 1), k)
    sigma = torch.randperm(e, generator=g, device="cuda")  # old id -> new id
    inv = torch.argsort(sigma)

    def run(ids, ww1, ww2):
        rt = sm.RoutingResult(ids, routing.p, torch.zeros((tokens, e), device="cuda"), renormalized=True,
                              validate=False)
        order = sm.compute_grouped_order(rt)
        y, ctx = sm.smoe_mlp_forward(x, ww1, ww2, rt, order)
        return y, sm.smoe_mlp_backward(ctx, dy)

    y0, g0 = run(routing.expert_idx, w1, w2)
    y1, g1 = run(sigma[routing.expert_idx].contiguous(), w1[inv].contiguous(), w2[inv].contiguous())
    assert torch.equal(y1, y0)
    assert torch.equal(g1.dx, g0.dx) and torch.equal(g1.dp, g0.dp)
    assert torch.equal(g1.dw1, g0.dw1[inv]) and torch.equal(g1.dw2, g0.dw2[inv])
