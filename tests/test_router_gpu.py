"""Router kernel (csrc/router.cu) vs the reference's gate outputs (tests/golden/gate.npz)."""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from conftest import load_golden
from gpu_util import np_of, t
from oracle import scattermlp_oracle as orc

pytestmark = pytest.mark.gpu


def test_topk_select_bit_exact_indices_on_reference_gates():
    g = load_golden("gate")
    for j in range(int(g["num_gate"])):
        pre = f"g{j}_"
        k, renorm = int(g[pre + "k"]), bool(g[pre + "renorm"])
        r = sm.topk_select(t(g[pre + "gate"]), k, renormalize=renorm)
        assert np.array_equal(r.expert_idx.cpu().numpy(), g[pre + "idx"])
        np.testing.assert_allclose(np_of(r.p), g[pre + "p"], rtol=1e-6, atol=1e-7)
        # fused softmax + top-k from logits
        r2 = sm.route(t(g[pre + "logits"]), k, renormalize=renorm)
        np.testing.assert_allclose(np_of(r2.gate_full), g[pre + "soft"], rtol=1e-6, atol=1e-8)
        assert np.array_equal(r2.expert_idx.cpu().numpy(), g[pre + "idx2"])
        np.testing.assert_allclose(np_of(r2.p), g[pre + "p2"], rtol=1e-6, atol=1e-7)
    r = sm.topk_select(t(g["tie_gate"]), 3, renormalize=False)
    assert np.array_equal(r.expert_idx.cpu().numpy(), g["tie_idx"])


def test_gate_backward_matches_reference():
    g = load_golden("gate")
    for j in range(int(g["num_gate"])):
        pre = f"g{j}_"
        k, renorm = int(g[pre + "k"]), bool(g[pre + "renorm"])
        gate = t(g[pre + "gate"])
        routing = sm.RoutingResult(t(g[pre + "idx"]), t(g[pre + "p"]), gate, renormalized=renorm, validate=False)
        dz = sm.gate_backward(routing, t(g[pre + "grad_p"]))
        np.testing.assert_allclose(np_of(dz), g[pre + "dz"], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("e,k", [(8, 2), (64, 8), (16, 4), (1000, 8), (3, 3)])
def test_router_large_random(e, k):
    rng = np.random.default_rng(e * 100 + k)
    logits = rng.standard_normal((20000, e)).astype(np.float32)
    logits[:100] = np.round(logits[:100])        # many exact ties
    gate = orc.softmax_rows(logits)
    r = sm.topk_select(t(gate), k)
    idx, p = orc.topk_routing(gate, k)
    assert np.array_equal(r.expert_idx.cpu().numpy(), idx)
    np.testing.assert_allclose(np_of(r.p), p, rtol=1e-6, atol=1e-7)
    r2 = sm.route(t(logits), k)
    np.testing.assert_allclose(np_of(r2.gate_full), gate, rtol=1e-6, atol=1e-9)
    assert np.array_equal(r2.expert_idx.cpu().numpy(), idx)


def test_fused_gate_topk_matches_reference_gate_vectors():
    """gate_topk(x, W_g, k) == topk_select(gate_forward(x, W_g), k) of the reference
    (tests/golden/gate.npz; router.py:119-151): bit-identical ids, gates and p to float32 rounding."""
    g = load_golden("gate")
    for j in range(int(g["num_gate"])):
        pre = f"g{j}_"
        k, renorm = int(g[pre + "k"]), bool(g[pre + "renorm"])
        for dtype in (torch.float32,):
            r = sm.gate_topk(t(g[pre + "x"]).to(dtype), t(g[pre + "wg"]), k, renormalize=renorm)
            assert np.array_equal(r.expert_idx.cpu().numpy(), g[pre + "idx"]), j
            np.testing.assert_allclose(np_of(r.gate_full), g[pre + "gate"], rtol=1e-6, atol=1e-8)
            np.testing.assert_allclose(np_of(r.p), g[pre + "p"], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("t_,d,e,k", [(32768, 4096, 8, 2), (4096, 4096, 64, 8), (3000, 2048, 16, 4), (257, 40, 5, 3)])
def test_fused_gate_topk_large(t_, d, e, k):
    """At BASELINE dims (C1: d_model=4096, E=8; C2/C4: E=64, k=8; C3: d_model=2048, E=16, k=4):
    float64 logits vs the oracle's gate_probs (f64 accumulate, router.py:121-122).  Indices
    are equal wherever the oracle's k-th and (k+1)-th gates differ by more than 2 float32
    ulps (order-of-summation differences in the f64 logits can flip a closer pair)."""
    rng = np.random.default_rng(t_ + e)
    x = rng.uniform(-1, 1, (t_, d)).astype(np.float32)
    wg = (rng.uniform(-1, 1, (d, e)) / np.sqrt(d)).astype(np.float32)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    xr = xb.float().numpy()
    r = sm.gate_topk(xb.cuda(), t(wg), k)
    gate = orc.gate_probs(xr, wg)
    idx, p = orc.topk_routing(gate, k)
    np.testing.assert_allclose(np_of(r.gate_full), gate, rtol=2e-6, atol=1e-9)
    srt = -np.sort(-gate, axis=1)
    clear = (srt[:, k - 1] - srt[:, k]) > 2 * np.spacing(srt[:, k - 1]) if k < e else np.ones(t_, bool)
    got = r.expert_idx.cpu().numpy()
    assert clear.mean() > 0.99
    assert np.array_equal(got[clear], idx[clear])
    np.testing.assert_allclose(np_of(r.p)[clear], p[clear], rtol=2e-6, atol=1e-7)
    # feeds K1 directly
    order = sm.compute_grouped_order(r)
    o_ref, off_ref = orc.compute_grouped_order(got, e)
    assert np.array_equal(order.o.cpu().numpy().astype(np.int64), o_ref)
