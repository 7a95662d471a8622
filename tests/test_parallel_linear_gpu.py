"""ParallelLinear forward/backward parity (parallel_linear.py:85-269) on the GPU."""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from conftest import load_golden
from gpu_util import np_of, order_of, rel_err, t

pytestmark = pytest.mark.gpu

LAYOUTS = {"s2g": sm.SCATTERED_TO_GROUPED, "g2s": sm.GROUPED_TO_SCATTERED,
           "s2s": sm.SCATTERED_TO_SCATTERED, "g2g": sm.GROUPED_TO_GROUPED}


def _case(g, j):
    pre = f"pl{j}_"
    order = order_of(g[pre + "idx"], int(g[pre + "E"]))
    p = t(g[pre + "p"]) if int(g[pre + "p_given"]) else None
    return pre, order, p, LAYOUTS[str(g[pre + "layout"])], int(g[pre + "fan_out"])


def test_golden_forward_backward_fp32():
    g = load_golden("parallel_linear")
    for j in range(int(g["num_pl"])):
        pre, order, p, layout, fan = _case(g, j)
        y, ctx = sm.parallel_linear_forward(t(g[pre + "x"]), t(g[pre + "w"]), order, p=p, fan_out=fan,
                                            layout=layout)
        np.testing.assert_allclose(np_of(y), g[pre + "y"], rtol=1e-5, atol=1e-6)
        gr = sm.parallel_linear_backward(ctx, t(g[pre + "dy"]))
        np.testing.assert_allclose(np_of(gr.dx), g[pre + "dx"], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(np_of(gr.dw), g[pre + "dw"], rtol=1e-5, atol=1e-5)
        if p is not None:
            np.testing.assert_allclose(np_of(gr.dp), g[pre + "dp"], rtol=1e-5, atol=1e-5)
        for got, name in ((gr.dx, "dx"), (gr.dw, "dw")):
            assert rel_err(got, g[pre + name]) <= 1e-4


def test_context_single_use_and_aliasing_rules():
    g = load_golden("parallel_linear")
    pre, order, p, layout, fan = _case(g, 4)   # a p-given case
    assert p is not None
    x, w = t(g[pre + "x"]), t(g[pre + "w"])
    y, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    dy = t(g[pre + "dy"])
    sm.parallel_linear_backward(ctx, dy)
    with pytest.raises(RuntimeError, match="consumed"):
        sm.parallel_linear_backward(ctx, dy)
    y, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    with pytest.raises(RuntimeError, match="alias"):
        sm.parallel_linear_backward(ctx, ctx.y_hat[: dy.shape[0]])
    # scratch slots must not alias each other
    y, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    n = order.num_slots
    buf = torch.empty((n, max(x.shape[1], w.shape[2])), device="cuda")
    ctx.scratch_grouped_dy = buf[:, : w.shape[2]]
    ctx.scratch_grouped_x = buf[:, : x.shape[1]]
    with pytest.raises(RuntimeError, match="alias"):
        sm.parallel_linear_backward(ctx, dy)


def test_seeded_scratch_is_bit_identical():
    """test_parallel_linear.py:175-200: seeded scratch gives identical results."""
    g = load_golden("parallel_linear")
    pre, order, p, layout, fan = _case(g, 4)
    x, w, dy = t(g[pre + "x"]), t(g[pre + "w"]), t(g[pre + "dy"])
    _, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    base = sm.parallel_linear_backward(ctx, dy)
    _, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    n = order.num_slots
    ctx.scratch_grouped_dy = torch.empty((n, w.shape[2]), device="cuda")
    ctx.scratch_grouped_x = torch.empty((n, w.shape[1]), device="cuda")
    other = sm.parallel_linear_backward(ctx, dy)
    assert torch.equal(base.dx, other.dx) and torch.equal(base.dw, other.dw) and torch.equal(base.dp, other.dp)


def test_autograd_function_matches_functional():
    g = load_golden("parallel_linear")
    pre, order, p, layout, fan = _case(g, 4)
    x = t(g[pre + "x"]).requires_grad_(True)
    w = t(g[pre + "w"]).requires_grad_(True)
    pp = p.clone().requires_grad_(True)
    y = sm.ParallelLinear.apply(x, w, order, fan, pp, layout.grouped_in, False)
    y.backward(t(g[pre + "dy"]))
    np.testing.assert_allclose(np_of(y), g[pre + "y"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np_of(x.grad), g[pre + "dx"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(np_of(w.grad), g[pre + "dw"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(np_of(pp.grad), g[pre + "dp"], rtol=1e-5, atol=1e-5)


def test_inference_combine_equals_training():
    """train == infer (test_parallel_linear.py:50-57), fp32 check mode."""
    g = load_golden("parallel_linear")
    pre, order, p, layout, fan = _case(g, 4)
    x, w = t(g[pre + "x"]), t(g[pre + "w"])
    y_train, _ = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout)
    y_inf, ctx = sm.parallel_linear_forward(x, w, order, p=p, fan_out=fan, layout=layout, training=False)
    assert ctx is None
    np.testing.assert_allclose(np_of(y_inf), np_of(y_train), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("shape", [(512, 4, 16, 512, 2048), (300, 2, 8, 136, 264), (64, 3, 5, 72, 520)])
def test_dp_epilogue_backward_bf16(shape, monkeypatch):
    """bf16 backward with combine weights and a scattered fan-out-1 input (the
    MoMHA output projection, moe_layers.py:446-449): dp computed inside the
    input-gradient GEMM's epilogue (<dY W^T, x> partials) and p moved to the x
    side of dW.  Against the oracle (bf16-rounded inputs, f64 accumulation) at
    the bf16 bar, and against the reference-ordered path (combine_grad_p)."""
    from oracle import scattermlp_oracle as orc
    from gpu_util import bf16_round
    t_tok, k, e, d_in, d_out = shape
    rng = np.random.default_rng(sum(shape))
    idx = np.stack([rng.permutation(e - 1)[:k] for _ in range(t_tok)])      # expert e-1 empty
    p = rng.uniform(0.05, 1.0, (t_tok, k)).astype(np.float32)
    n = t_tok * k
    x = bf16_round(rng.uniform(-1, 1, (n, d_in)))
    w = bf16_round(rng.uniform(-1, 1, (e, d_in, d_out)) / np.sqrt(d_in))
    dy = bf16_round(rng.uniform(-1, 1, (t_tok, d_out)))
    o, off = orc.compute_grouped_order(idx, e)
    want_y, y_hat = orc.pl_forward(x.astype(np.float64), w.astype(np.float64), o, off, p.astype(np.float64), 1,
                                   False, False)
    want = orc.pl_backward(x.astype(np.float64), w.astype(np.float64), o, off, p.astype(np.float64), 1, False,
                           False, y_hat, dy.astype(np.float64))
    import sys
    plmod = sys.modules["paper_2403_08245_b200.parallel_linear"]   # sm.parallel_linear is the function
    order = order_of(idx, e)
    got = {}
    for mode in (True, False):
        monkeypatch.setattr(plmod, "_DP_EPILOGUE", mode)
        y, ctx = sm.parallel_linear_forward(t(x, torch.bfloat16), t(w, torch.bfloat16), order, p=t(p), fan_out=1,
                                            layout=sm.SCATTERED_TO_SCATTERED)
        gr = sm.parallel_linear_backward(ctx, t(dy, torch.bfloat16))
        got[mode] = gr
        assert rel_err(y, want_y) <= 2e-2
        for val, ref, name in ((gr.dx, want[0], "dx"), (gr.dw, want[1], "dw"), (gr.dp, want[2], "dp")):
            assert rel_err(val, ref) <= 2e-2, (mode, name, rel_err(val, ref))
        assert float(gr.dw[e - 1].float().abs().max()) == 0.0
    assert rel_err(got[True].dp, np_of(got[False].dp)) <= 1e-2


@pytest.mark.parametrize("seed", range(16))
def test_bf16_random_shapes_vs_oracle(seed, monkeypatch):
    """Seeded random sweep of ParallelLinear forward + backward in bf16: every
    layout, with and without combine weights, fan-out 1 or k on scattered
    inputs, and the grouped-Y_hat / dp-epilogue flows on and off, against the
    oracle (f64 on the bf16-rounded inputs) at the bf16 bar."""
    import sys
    from oracle import scattermlp_oracle as orc
    from gpu_util import bf16_round
    plmod = sys.modules["paper_2403_08245_b200.parallel_linear"]
    rng = np.random.default_rng(3000 + seed)
    e = int(rng.choice([1, 3, 8, 16, 64]))
    k = int(rng.integers(1, min(e, 4) + 1))
    tokens = int(rng.choice([1, 7, 130, 600]))
    d_in, d_out = int(8 * rng.integers(1, 50)), int(8 * rng.integers(1, 50))
    layout = list(LAYOUTS.values())[seed % 4]
    with_p = bool((seed // 4) % 2)
    if with_p:      # combine weights need scattered kernel output (parallel_linear.py:118-119)
        layout = sm.GROUPED_TO_SCATTERED if layout.grouped_in else sm.SCATTERED_TO_SCATTERED
    fan = 1 if layout.grouped_in else int(rng.choice([1, k]))
    monkeypatch.setattr(plmod, "_GROUPED_YHAT", bool(seed % 3))
    monkeypatch.setattr(plmod, "_DP_EPILOGUE", bool(seed % 5))
    idx = np.stack([rng.permutation(e)[:k] for _ in range(tokens)])
    n = tokens * k
    x = bf16_round(rng.uniform(-1, 1, (n if (layout.grouped_in or fan == 1) else n // fan, d_in)))
    w = bf16_round(rng.uniform(-1, 1, (e, d_in, d_out)) / np.sqrt(d_in))
    p = rng.uniform(0.05, 1.0, (tokens, k)).astype(np.float32) if with_p else None
    dy = bf16_round(rng.uniform(-1, 1, ((tokens if with_p else n), d_out)))
    o, off = orc.compute_grouped_order(idx, e)
    p64 = None if p is None else p.astype(np.float64)
    want_y, y_hat = orc.pl_forward(x.astype(np.float64), w.astype(np.float64), o, off, p64, fan,
                                   layout.grouped_in, layout.grouped_out)
    want = orc.pl_backward(x.astype(np.float64), w.astype(np.float64), o, off, p64, fan, layout.grouped_in,
                           layout.grouped_out and not with_p, y_hat, dy.astype(np.float64))
    order = order_of(idx, e)
    y, ctx = sm.parallel_linear_forward(t(x, torch.bfloat16), t(w, torch.bfloat16), order,
                                        p=None if p is None else t(p), fan_out=fan, layout=layout)
    gr = sm.parallel_linear_backward(ctx, t(dy, torch.bfloat16))
    case = (tokens, k, e, d_in, d_out, layout, with_p, fan)
    assert rel_err(y, want_y) <= 2e-2, case
    assert rel_err(gr.dx, want[0]) <= 2e-2, ("dx", case)
    assert rel_err(gr.dw, want[1]) <= 2e-2, ("dw", case)
    if with_p:
        absdot = (np.abs(dy).astype(np.float64)[:, None, :] * np.abs(y_hat).reshape(tokens, k, d_out)).sum(-1)
        err = np.abs(np_of(gr.dp).astype(np.float64) - want[2])
        assert np.all(err <= 2e-2 * absdot + 1e-6), ("dp", case)
