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
