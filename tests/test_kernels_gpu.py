"""scatter2scatter / group / group_xty / scatter_combine parity on the GPU.

fp32 check mode (engine=simt): the reference's elementwise tolerance
(rtol 1e-5, test_kernels.py:65) plus an absolute floor for fp32-vs-f64
accumulation, and <= 1e-4 relative Frobenius (north_star).
bf16 (engine auto -> tcgen05 when built): oracle fed the bf16-rounded inputs,
relative Frobenius error <= 2e-2 per tensor (north_star).
"""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from conftest import load_golden
from gpu_util import bf16_round, np_of, order_of, rel_err, t
from oracle import scattermlp_oracle as orc

pytestmark = pytest.mark.gpu

LAYOUTS = {"s2g": sm.SCATTERED_TO_GROUPED, "g2s": sm.GROUPED_TO_SCATTERED,
           "s2s": sm.SCATTERED_TO_SCATTERED, "g2g": sm.GROUPED_TO_GROUPED}
FP32_RTOL, FP32_ATOL = 1e-5, 1e-6
ENGINES = ["simt", "auto"]


def test_golden_scatter2scatter_fp32():
    g = load_golden("kernels")
    for j in range(int(g["num_s2s"])):
        pre = f"s2s{j}_"
        order = order_of(g[pre + "idx"], int(g[pre + "E"]))
        y = sm.scatter2scatter(t(g[pre + "x"]), t(g[pre + "w"]), order, int(g[pre + "fan_out"]),
                               LAYOUTS[str(g[pre + "layout"])], transpose_w=bool(g[pre + "transpose"]))
        np.testing.assert_allclose(np_of(y), g[pre + "y"], rtol=FP32_RTOL, atol=FP32_ATOL, err_msg=str(j))
        assert rel_err(y, g[pre + "y"]) <= 1e-4


def test_golden_group_xty_combine_fp32():
    g = load_golden("kernels")
    order = order_of(g["grp_idx"], 5)
    np.testing.assert_array_equal(np_of(sm.group(t(g["grp_x"]), order, fan_out=2)), g["grp_plain"])
    got = sm.group(t(g["grp_x"]), order, weights=t(g["grp_p"].reshape(-1)), fan_out=2)
    np.testing.assert_allclose(np_of(got), g["grp_weighted"], rtol=1e-6, atol=1e-7)
    order2 = order_of(g["xty_idx"], 6)
    dw = sm.group_xty(t(g["xty_x"]), t(g["xty_y"]), order2)
    np.testing.assert_allclose(np_of(dw), g["xty_dw"], rtol=FP32_RTOL, atol=FP32_ATOL)
    assert float(dw[5].abs().max()) == 0.0  # skip_one: expert 5 has an empty bin
    sc = sm.scatter_combine(t(g["grp_x"]), t(g["sc_w"]), order, 2, t(g["grp_p"].reshape(-1)), 2, False)
    np.testing.assert_allclose(np_of(sc), g["sc_y"], rtol=FP32_RTOL, atol=FP32_ATOL)


def _problem(rng, tokens, k, e, d_in, d_out, layout, transpose, flavor="gate"):
    if flavor == "all_to_one":
        idx = np.tile(np.arange(k), (tokens, 1))
    elif flavor == "skip_one":
        idx = np.stack([rng.permutation(e - 1)[:k] for _ in range(tokens)])
    else:
        idx = np.stack([rng.permutation(e)[:k] for _ in range(tokens)])
    rows = tokens * k if layout.grouped_in else tokens
    fan_out = 1 if layout.grouped_in else k
    x = rng.uniform(-1, 1, (rows, d_in)).astype(np.float32)
    shape = (e, d_out, d_in) if transpose else (e, d_in, d_out)
    w = (rng.uniform(-1, 1, shape) / np.sqrt(d_in)).astype(np.float32)
    return idx, x, w, fan_out


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("lname", list(LAYOUTS))
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("flavor", ["gate", "all_to_one", "skip_one"])
def test_bf16_layouts_vs_oracle(engine, lname, transpose, flavor):
    """Tile-sized and ragged shapes, bf16 storage, fp32 accumulate."""
    rng = np.random.default_rng(hash((lname, transpose, flavor)) % 2**32)
    layout = LAYOUTS[lname]
    for tokens, k, e, d_in, d_out in [(300, 2, 6, 256, 512), (1000, 2, 8, 128, 256), (77, 3, 5, 64, 192)]:
        idx, x, w, fan_out = _problem(rng, tokens, k, e, d_in, d_out, layout, transpose, flavor)
        xb, wb = bf16_round(x), bf16_round(w)
        o, off = orc.compute_grouped_order(idx, e)
        want = orc.scatter2scatter(xb, wb, o, off, fan_out, layout.grouped_in, layout.grouped_out, transpose)
        order = order_of(idx, e)
        y = sm.scatter2scatter(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out, layout,
                               transpose_w=transpose, engine=engine)
        assert y.dtype == torch.bfloat16
        assert rel_err(y, want) <= 2e-2, (tokens, k, e, d_in, d_out)


@pytest.mark.parametrize("engine", ENGINES)
def test_layout_consistency_bit_identical(engine):
    """grouped-out composed with the inverse permutation == scattered-out (test_acceptance.py:349-381)."""
    rng = np.random.default_rng(6)
    for dtype in (torch.float32, torch.bfloat16):
        idx, x, w, fan_out = _problem(rng, 500, 2, 8, 128, 256, sm.SCATTERED_TO_GROUPED, False)
        order = order_of(idx, 8)
        xt, wt = t(x, dtype), t(w, dtype)
        grouped = sm.scatter2scatter(xt, wt, order, fan_out, sm.SCATTERED_TO_GROUPED, engine=engine)
        scattered = sm.scatter2scatter(xt, wt, order, fan_out, sm.SCATTERED_TO_SCATTERED, engine=engine)
        assert torch.equal(grouped[order.inverse().long()], scattered)


@pytest.mark.parametrize("engine", ENGINES)
def test_out_reuse_and_determinism_bit_identical(engine):
    rng = np.random.default_rng(8)
    idx, x, w, _ = _problem(rng, 400, 2, 8, 128, 128, sm.GROUPED_TO_SCATTERED, False)
    order = order_of(idx, 8)
    xt, wt = t(x, torch.bfloat16), t(w, torch.bfloat16)
    fresh = sm.scatter2scatter(xt, wt, order, 1, sm.GROUPED_TO_SCATTERED, engine=engine)
    out = torch.full_like(fresh, float("nan"))
    reused = sm.scatter2scatter(xt, wt, order, 1, sm.GROUPED_TO_SCATTERED, out=out, engine=engine)
    assert reused.data_ptr() == out.data_ptr()
    assert torch.equal(fresh, reused)
    again = sm.scatter2scatter(xt, wt, order, 1, sm.GROUPED_TO_SCATTERED, engine=engine)
    assert torch.equal(fresh, again)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("flavor", ["gate", "all_to_one", "skip_one"])
def test_group_xty_bf16(engine, flavor):
    rng = np.random.default_rng(11)
    e = 6
    for n_tok, k, d_in, d_out in [(600, 2, 128, 256), (333, 2, 256, 128), (50, 1, 64, 64)]:
        idx, _, _, _ = _problem(rng, n_tok, k, e, 8, 8, sm.SCATTERED_TO_GROUPED, False, flavor)
        order = order_of(idx, e)
        n = n_tok * k
        xg = bf16_round(rng.uniform(-1, 1, (n, d_in)).astype(np.float32))
        yg = bf16_round(rng.uniform(-1, 1, (n, d_out)).astype(np.float32))
        o, off = orc.compute_grouped_order(idx, e)
        want = orc.group_xty(xg, yg, off)
        dw = sm.group_xty(t(xg, torch.bfloat16), t(yg, torch.bfloat16), order, engine=engine)
        assert rel_err(dw, want) <= 2e-2
        counts = np.diff(off)
        for ee in np.nonzero(counts == 0)[0]:
            assert float(dw[ee].float().abs().max()) == 0.0


@pytest.mark.parametrize("act", ["gelu", "relu", "silu"])
@pytest.mark.parametrize("engine", ENGINES)
def test_fused_activation_epilogues(act, engine):
    rng = np.random.default_rng(12)
    idx, x, w, fan_out = _problem(rng, 300, 2, 8, 128, 256, sm.SCATTERED_TO_GROUPED, False)
    xb, wb = bf16_round(x), bf16_round(w)
    order = order_of(idx, 8)
    o, off = orc.compute_grouped_order(idx, 8)
    pre = torch.empty((600, 256), dtype=torch.bfloat16, device="cuda")
    h = torch.empty_like(pre)
    sm.scatter2scatter(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, 2, sm.SCATTERED_TO_GROUPED,
                       out=pre, activation=act, act_out=h, engine=engine)
    want_pre = orc.scatter2scatter(xb, wb, o, off, 2, False, True)
    assert rel_err(pre, want_pre) <= 2e-2
    want_h = orc.act(np_of(pre), act)            # act of the stored (rounded) pre-activation
    assert rel_err(h, want_h) <= 1e-2
    # act-grad epilogue on a G2G transposed product
    dyg = bf16_round(rng.uniform(-1, 1, (600, 128)).astype(np.float32))
    w2 = bf16_round((rng.uniform(-1, 1, (8, 256, 128)) / 16).astype(np.float32))
    dh = torch.empty_like(pre)
    sm.scatter2scatter(t(dyg, torch.bfloat16), t(w2, torch.bfloat16), order, 1, sm.GROUPED_TO_GROUPED,
                       transpose_w=True, out=dh, activation=act, act_grad_of=pre, engine=engine)
    want_dh = orc.scatter2scatter(dyg, w2, o, off, 1, True, True, transpose_w=True) * orc.act_grad(np_of(pre), act)
    assert rel_err(dh, want_dh) <= 2e-2


def test_row_kernels_bf16():
    rng = np.random.default_rng(13)
    tokens, k, d = 1000, 2, 512
    p = rng.random((tokens, k)).astype(np.float32)
    y_hat = bf16_round(rng.uniform(-1, 1, (tokens * k, d)).astype(np.float32))
    dy = bf16_round(rng.uniform(-1, 1, (tokens, d)).astype(np.float32))
    yh = t(y_hat, torch.bfloat16)
    y = sm.kernels.combine(t(p), yh)
    assert rel_err(y, orc.combine(p, y_hat)) <= 1e-2
    dp = sm.kernels.combine_grad_p(t(dy, torch.bfloat16), yh, tokens, k)
    assert rel_err(dp, orc.combine_grad_p(dy, y_hat, tokens, k)) <= 1e-4
    dx = sm.kernels.fanout_reduce(yh, k)
    assert rel_err(dx, orc.fanout_reduce(y_hat, k)) <= 1e-2


@pytest.mark.parametrize("grouped_in", [False, True])
@pytest.mark.parametrize("flavor", ["gate", "all_to_one", "skip_one"])
def test_scatter_combine_bf16_tcgen05(grouped_in, flavor):
    """Inference combine on the tensor cores (kernels.py:242-286): the GEMM
    epilogue scales each slot row by p and reduces it into the fp32 token row."""
    rng = np.random.default_rng(hash(("combine", grouped_in, flavor)) % 2**32)
    layout = sm.GROUPED_TO_SCATTERED if grouped_in else sm.SCATTERED_TO_SCATTERED
    for tokens, k, e, d_in, d_out in [(300, 2, 6, 256, 512), (1000, 4, 8, 128, 256), (77, 3, 5, 64, 200)]:
        idx, x, w, fan_out = _problem(rng, tokens, k, e, d_in, d_out, layout, False, flavor)
        p = rng.uniform(0.05, 1.0, (tokens, k)).astype(np.float32)
        xb, wb = bf16_round(x), bf16_round(w)
        o, off = orc.compute_grouped_order(idx, e)
        want = orc.scatter_combine(xb, wb, o, off, fan_out, p.reshape(-1), k, grouped_in)
        order = order_of(idx, e)
        y = sm.scatter_combine(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out,
                               t(p.reshape(-1)), k, grouped_in, engine="tcgen05")
        assert y.dtype == torch.bfloat16 and tuple(y.shape) == (tokens, d_out)
        assert rel_err(y, want) <= 2e-2, (tokens, k, rel_err(y, want))
        # same as the SIMT engine within bf16 rounding
        ys = sm.scatter_combine(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out,
                                t(p.reshape(-1)), k, grouped_in, engine="simt")
        assert rel_err(y, np_of(ys)) <= 1e-2
        # default (GEMM to slot rows + token-major combine): deterministic
        y2 = sm.scatter_combine(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out,
                                t(p.reshape(-1)), k, grouped_in, engine="tcgen05")
        assert torch.equal(y, y2)
        # the fused combine epilogue (SMOE_COMBINE_FUSED=1): p-scaled rows reduced
        # into fp32 token rows in L2; k <= 2 is bit-reproducible (two additions
        # into a zeroed row commute), k > 2 lands in completion order
        prev = sm.kernels._COMBINE_FUSED
        sm.kernels._COMBINE_FUSED = "1"
        try:
            yf = sm.scatter_combine(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out,
                                    t(p.reshape(-1)), k, grouped_in, engine="tcgen05")
            yf2 = sm.scatter_combine(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out,
                                     t(p.reshape(-1)), k, grouped_in, engine="tcgen05")
        finally:
            sm.kernels._COMBINE_FUSED = prev
        assert rel_err(yf, want) <= 2e-2
        if k <= 2:
            assert torch.equal(yf, yf2)


def test_inference_mlp_uses_tcgen05_combine():
    """smoe_mlp_forward(training=False) at a C1-like shape: the layer-2 combine
    runs on the tensor cores and matches the training path's combine."""
    g = torch.Generator(device="cuda").manual_seed(5)
    tokens, d, de, e, k = 4096, 1024, 2048, 8, 2
    x = (torch.rand((tokens, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    w1 = ((torch.rand((e, d, de), generator=g, device="cuda") * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    w2 = ((torch.rand((e, de, d), generator=g, device="cuda") * 2 - 1) / de ** 0.5).to(torch.bfloat16)
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    from paper_2403_08245_b200.launch_timer import LaunchTimer
    with LaunchTimer() as lt:
        y_inf, _ = sm.smoe_mlp_forward(x, w1, w2, routing, order, training=False)
    labels = list(lt.summary())
    assert any(lab.startswith("scatter2scatter G->S") for lab in labels), labels
    y_tr, _ = sm.smoe_mlp_forward(x, w1, w2, routing, order, training=True)
    assert rel_err(y_inf, np_of(y_tr)) <= 1e-2
    prev = sm.kernels._COMBINE_FUSED
    sm.kernels._COMBINE_FUSED = "1"
    try:
        with LaunchTimer() as lt:
            y_fused, _ = sm.smoe_mlp_forward(x, w1, w2, routing, order, training=False)
    finally:
        sm.kernels._COMBINE_FUSED = prev
    assert any(lab.startswith("scatter_combine") for lab in lt.summary())
    assert rel_err(y_fused, np_of(y_tr)) <= 1e-2


@pytest.mark.parametrize("engine", ["auto", "simt"])
@pytest.mark.parametrize("flavor", ["gate", "all_to_one", "skip_one"])
@pytest.mark.parametrize("grouped", [(False, True), (True, False), (False, False)])
def test_group_xty_scattered_matches_group_then_xty(engine, flavor, grouped):
    """Gathered weight-gradient operands == the reference's group() copies + group_xty
    (bit-identical on the tensor cores: same rows land in the same smem slots)."""
    xg_flag, yg_flag = grouped
    rng = np.random.default_rng(hash(("xtys", flavor, grouped)) % 2**32)
    dt = torch.bfloat16 if engine == "auto" else torch.float32
    for tokens, k, e, d_in, d_out in [(300, 2, 6, 256, 512), (1000, 3, 8, 136, 264), (77, 1, 5, 64, 192),
                                      (4096, 2, 8, 512, 256)]:
        idx, _, _, _ = _problem(rng, tokens, k, e, 8, 8, sm.SCATTERED_TO_GROUPED, False, flavor)
        n = tokens * k
        fx, fy = (1 if xg_flag else k), (1 if yg_flag else 1)
        x = bf16_round(rng.uniform(-1, 1, (n if xg_flag else n // fx, d_in)).astype(np.float32))
        y = bf16_round(rng.uniform(-1, 1, (n if yg_flag else n // fy, d_out)).astype(np.float32))
        order = order_of(idx, e)
        xt, yt = t(x, dt), t(y, dt)
        got = sm.kernels.group_xty_scattered(xt, yt, order, x_fan_out=fx, y_fan_out=fy, x_grouped=xg_flag,
                                             y_grouped=yg_flag, engine=engine)
        xb = xt if xg_flag else sm.group(xt, order, fan_out=fx)
        yb = yt if yg_flag else sm.group(yt, order, fan_out=fy)
        want = sm.group_xty(xb, yb, order, engine=engine)
        if engine == "auto":
            assert torch.equal(got, want), (tokens, k, e)
        else:
            o, off = orc.compute_grouped_order(idx, e)
            xo = x if xg_flag else x[o // fx]
            yo = y if yg_flag else y[o // fy]
            ref = orc.group_xty(xo, yo, off)
            # fp32 sums of up to ~3000 products of magnitude <= 1 vs f64
            np.testing.assert_allclose(np_of(got), ref, rtol=FP32_RTOL, atol=1e-4)
            assert rel_err(got, ref) <= 1e-5
        if flavor == "skip_one":
            assert float(got[e - 1].abs().max()) == 0.0


@pytest.mark.parametrize("k", [1, 2, 3, 8])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_group_token_major_equals_grouped_walk(k, weighted, dtype):
    """group() walking source rows (smoe_group_inv) == walking grouped positions."""
    rng = np.random.default_rng(k * 7 + weighted)
    tokens, e, d = 777, 9, 264
    idx = np.stack([rng.permutation(e)[:k] for _ in range(tokens)])
    order = order_of(idx, e)
    x = t(rng.uniform(-1, 1, (tokens, d)).astype(np.float32), dtype)
    w = t(rng.uniform(0, 1, tokens * k).astype(np.float32)) if weighted else None
    got = sm.group(x, order, weights=w, fan_out=k)
    prev = sm.kernels._GROUP_BY_TOKEN
    sm.kernels._GROUP_BY_TOKEN = False
    try:
        want = sm.group(x, order, weights=w, fan_out=k)
    finally:
        sm.kernels._GROUP_BY_TOKEN = prev
    assert torch.equal(got, want)


def test_bf16_unsupported_shape_is_refused():
    """bf16 with d_out % 8 != 0: NotImplementedError (SMOE_ENOTSUP), no SIMT fallback;
    the same call with engine='simt' (explicit cross-check) still runs."""
    rng = np.random.default_rng(5)
    idx = np.stack([rng.permutation(4)[:2] for _ in range(16)]).astype(np.int64)
    order = order_of(idx, 4)
    x = t(rng.standard_normal((16, 16)).astype(np.float32), torch.bfloat16)
    w = t(rng.standard_normal((4, 16, 12)).astype(np.float32), torch.bfloat16)
    with pytest.raises(NotImplementedError, match="no SIMT fallback"):
        sm.scatter2scatter(x, w, order, 2, sm.SCATTERED_TO_GROUPED)
    y = sm.scatter2scatter(x, w, order, 2, sm.SCATTERED_TO_GROUPED, engine="simt")
    o_ref, off_ref = orc.compute_grouped_order(idx, 4)
    want = orc.scatter2scatter(np_of(x), np_of(w), o_ref, off_ref, 2, False, True)
    assert rel_err(y, want) < 2e-2


def test_fp32_check_mode_accumulates_in_64_bit():
    """The check mode rounds once from a 64-bit sum (core_tensor.py:1-7): the
    reference's known case [2^24, 1, -2^24] . 1 = 1 (test_core_tensor.py:32-37),
    which fp32 accumulation gets wrong (0)."""
    order = order_of(np.zeros((1, 1), dtype=np.int64), 1)
    x = t(np.array([[2.0 ** 24, 1.0, -(2.0 ** 24)]], dtype=np.float32))
    w = t(np.ones((1, 3, 1), dtype=np.float32))
    y = sm.scatter2scatter(x, w, order, 1, sm.SCATTERED_TO_SCATTERED)
    assert float(y[0, 0]) == 1.0
    dw = sm.group_xty(t(np.array([[2.0 ** 24], [1.0], [-(2.0 ** 24)]], dtype=np.float32)),
                      t(np.ones((3, 1), dtype=np.float32)), order_of(np.zeros((3, 1), dtype=np.int64), 1))
    assert float(dw[0, 0, 0]) == 1.0


@pytest.mark.parametrize("k,d,dt", [(1, 264, torch.bfloat16), (2, 264, torch.bfloat16), (3, 264, torch.bfloat16),
                                    (4, 264, torch.bfloat16), (8, 264, torch.bfloat16), (2, 130, torch.bfloat16),
                                    (4, 96, torch.float32), (3, 33, torch.float64)])
def test_grouped_row_reductions_match_slot_order(k, d, dt):
    """fanout_reduce / combine / combine_grad_p over grouped rows (through the
    inverse permutation) are bit-identical to the slot-ordered kernels
    (vectorised and scalar paths, bf16 / fp32 / fp64 storage)."""
    g = torch.Generator(device="cuda").manual_seed(k)
    tokens, e = 777, 8
    routing = sm.topk_select(torch.softmax(torch.randn(tokens, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    slots = (torch.rand((tokens * k, d), device="cuda", generator=g) * 2 - 1).to(dt)
    grouped = slots[order.o.long()]                     # row i = slot o[i]
    inv = order.inverse()
    assert torch.equal(sm.kernels.fanout_reduce(grouped, k, inverse=inv), sm.kernels.fanout_reduce(slots, k))
    p = routing.p.float()
    assert torch.equal(sm.kernels.combine(p, grouped, inverse=inv), sm.kernels.combine(p, slots))
    dy = (torch.rand((tokens, d), device="cuda", generator=g) * 2 - 1).to(dt)
    assert torch.equal(sm.kernels.combine_grad_p(dy, grouped, tokens, k, inverse=inv),
                       sm.kernels.combine_grad_p(dy, slots, tokens, k))


def _random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    e = int(rng.choice([1, 2, 3, 7, 8, 16, 33, 64, 128]))
    k = int(rng.integers(1, min(e, 8) + 1))
    tokens = int(rng.choice([1, 2, 5, 31, 129, 257, 700, 1500]))
    d_in = int(8 * rng.integers(1, 70))
    d_out = int(8 * rng.integers(1, 70))
    d_in = 8 if seed in (3, 10) else d_in      # one 8-wide k-block
    d_out = 8 if seed in (7, 16) else d_out    # one 8-wide output column block
    return rng, tokens, k, e, d_in, d_out


@pytest.mark.parametrize("seed", range(24))
def test_bf16_random_shapes_vs_oracle(seed):
    """Seeded random sweep over expert counts (1..128), fan-out (1..8), token
    counts down to one and widths down to 8 (sub-tile K and N, ragged bins):
    every layout and transpose flag, plus group_xty, against the oracle."""
    rng, tokens, k, e, d_in, d_out = _random_case(seed)
    lname = list(LAYOUTS)[seed % 4]
    layout, transpose = LAYOUTS[lname], bool((seed // 4) % 2)
    flavor = ["gate", "all_to_one", "skip_one"][seed % 3]
    if flavor == "skip_one" and k >= e:
        flavor = "gate"
    idx, x, w, fan_out = _problem(rng, tokens, k, e, d_in, d_out, layout, transpose, flavor)
    xb, wb = bf16_round(x), bf16_round(w)
    o, off = orc.compute_grouped_order(idx, e)
    want = orc.scatter2scatter(xb, wb, o, off, fan_out, layout.grouped_in, layout.grouped_out, transpose)
    order = order_of(idx, e)
    y = sm.scatter2scatter(t(xb, torch.bfloat16), t(wb, torch.bfloat16), order, fan_out, layout,
                           transpose_w=transpose)
    assert rel_err(y, want) <= 2e-2, (lname, transpose, tokens, k, e, d_in, d_out)
    xg = bf16_round(rng.uniform(-1, 1, (tokens * k, d_in)).astype(np.float32))
    yg = bf16_round(rng.uniform(-1, 1, (tokens * k, d_out)).astype(np.float32))
    dw = sm.group_xty(t(xg, torch.bfloat16), t(yg, torch.bfloat16), order)
    want_dw = orc.group_xty(xg, yg, off)
    assert rel_err(dw, want_dw) <= 2e-2, ("xty", tokens, k, e, d_in, d_out)
    counts = np.diff(off)
    for ex in np.flatnonzero(counts == 0):
        assert float(dw[ex].float().abs().max()) == 0.0
