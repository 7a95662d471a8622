"""Pin the CPU oracle (oracle/scattermlp_oracle.py) to the reference's own outputs.

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Integer routing work must match bit for bit;
float work within the reference's own forward tolerance (rtol 1e-5, atol 1e-7,
test_acceptance.py:62-63) — the oracle restates the same f64-accumulate
arithmetic, so in practice it matches to the last bit or one ulp.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import scattermlp_oracle as orc

RTOL, ATOL = 1e-5, 1e-7


def test_routing_known_answers():
    g = load_golden("routing")
    for i in range(int(g["num_kats"])):
        o, off = orc.compute_grouped_order(g[f"kat{i}_idx"], int(g[f"kat{i}_E"]))
        assert np.array_equal(o, g[f"kat{i}_o"])
        assert np.array_equal(off, g[f"kat{i}_off"])
    # the literal vectors of test_router.py:58-77 and SPEC.md:131
    assert orc.compute_grouped_order(np.array([[1], [0], [1]]), 2)[0].tolist() == [1, 0, 2]
    assert orc.compute_grouped_order(np.array([[0, 2], [1, 0]]), 3)[0].tolist() == [0, 3, 2, 1]
    assert orc.compute_grouped_order(np.array([[0, 2], [1, 0]]), 3)[1].tolist() == [0, 2, 3, 4]
    assert orc.compute_grouped_order(np.array([[0, 1], [2, 0]]), 3)[0].tolist() == [0, 3, 1, 2]
    assert orc.compute_grouped_order(np.array([[0, 1], [1, 0]]), 2)[0].tolist() == [0, 3, 1, 2]


def test_routing_cases_bit_exact():
    g = load_golden("routing")
    for j in range(int(g["num_cases"])):
        o, off = orc.compute_grouped_order(g[f"case{j}_idx"], int(g[f"case{j}_E"]))
        assert np.array_equal(o, g[f"case{j}_o"]), j
        assert np.array_equal(off, g[f"case{j}_off"]), j
        inv = orc.inverse(o)
        assert np.array_equal(o[inv], np.arange(o.size))


LAYOUTS = {"s2g": (False, True), "g2s": (True, False), "s2s": (False, False), "g2g": (True, True)}


def test_scatter2scatter_all_layouts():
    g = load_golden("kernels")
    for j in range(int(g["num_s2s"])):
        pre = f"s2s{j}_"
        gin, gout = LAYOUTS[str(g[pre + "layout"])]
        o, off = orc.compute_grouped_order(g[pre + "idx"], int(g[pre + "E"]))
        y = orc.scatter2scatter(g[pre + "x"], g[pre + "w"], o, off, int(g[pre + "fan_out"]), gin, gout,
                                bool(g[pre + "transpose"]))
        np.testing.assert_allclose(y, g[pre + "y"], rtol=RTOL, atol=ATOL)


def test_group_xty_combine():
    g = load_golden("kernels")
    o, off = orc.compute_grouped_order(g["grp_idx"], 5)
    np.testing.assert_array_equal(orc.group(g["grp_x"], o, fan_out=2), g["grp_plain"])
    np.testing.assert_allclose(orc.group(g["grp_x"], o, g["grp_p"].reshape(-1), 2), g["grp_weighted"],
                               rtol=RTOL, atol=ATOL)
    o2, off2 = orc.compute_grouped_order(g["xty_idx"], 6)
    np.testing.assert_allclose(orc.group_xty(g["xty_x"], g["xty_y"], off2), g["xty_dw"], rtol=RTOL, atol=ATOL)
    sc = orc.scatter_combine(g["grp_x"], g["sc_w"], o, off, 2, g["grp_p"].reshape(-1), 2, False)
    np.testing.assert_allclose(sc, g["sc_y"], rtol=RTOL, atol=ATOL)


def test_parallel_linear_forward_backward():
    g = load_golden("parallel_linear")
    for j in range(int(g["num_pl"])):
        pre = f"pl{j}_"
        gin, gout = LAYOUTS[str(g[pre + "layout"])]
        e = int(g[pre + "E"])
        o, off = orc.compute_grouped_order(g[pre + "idx"], e)
        p = g[pre + "p"] if int(g[pre + "p_given"]) else None
        fan = int(g[pre + "fan_out"])
        y, y_hat = orc.pl_forward(g[pre + "x"], g[pre + "w"], o, off, p, fan, gin, gout)
        np.testing.assert_allclose(y, g[pre + "y"], rtol=RTOL, atol=ATOL)
        dx, dw, dp = orc.pl_backward(g[pre + "x"], g[pre + "w"], o, off, p, fan, gin, gout if p is None else False,
                                     y_hat, g[pre + "dy"])
        np.testing.assert_allclose(dx, g[pre + "dx"], rtol=RTOL, atol=1e-6)
        np.testing.assert_allclose(dw, g[pre + "dw"], rtol=RTOL, atol=1e-6)
        if p is not None:
            np.testing.assert_allclose(dp, g[pre + "dp"], rtol=RTOL, atol=1e-6)


def test_smoe_mlp_forward_backward():
    g = load_golden("mlp")
    for j in range(int(g["num_mlp"])):
        pre = f"mlp{j}_"
        act = str(g[pre + "act"])
        y, st = orc.smoe_mlp_forward(g[pre + "x"], g[pre + "w1"], g[pre + "w2"], g[pre + "idx"], g[pre + "p"],
                                     int(g[pre + "E"]), act)
        np.testing.assert_allclose(y, g[pre + "y"], rtol=RTOL, atol=ATOL)
        np.testing.assert_allclose(y, g[pre + "y_naive"], rtol=RTOL, atol=1e-6)
        dx, dw1, dw2, dp = orc.smoe_mlp_backward(g[pre + "x"], g[pre + "w1"], g[pre + "w2"], g[pre + "p"], st,
                                                 g[pre + "dy"], act)
        for got, name in ((dx, "dx"), (dw1, "dw1"), (dw2, "dw2"), (dp, "dp")):
            np.testing.assert_allclose(got, g[pre + name], rtol=RTOL, atol=1e-6, err_msg=f"{j}:{name}")


def test_momha_forward_backward():
    """The attention-layer restatement (moe_layers.py:270-482) against the reference's outputs."""
    g = load_golden("momha")
    seq_len, d_head = int(g["seq_len"]), 4
    y, st = orc.momha_forward(g["x"], g["wq"], g["wk"], g["wv"], g["wo"], g["idx"], g["p"], 3, seq_len, d_head)
    np.testing.assert_allclose(y, g["y"], rtol=RTOL, atol=ATOL)
    got = orc.momha_backward(g["x"], g["wq"], g["wk"], g["wv"], g["wo"], g["p"], st, g["dy"])
    for val, name in zip(got, ("dx", "dwq", "dwk", "dwv", "dwo", "dp")):
        np.testing.assert_allclose(val, g[name], rtol=RTOL, atol=1e-6, err_msg=name)


@pytest.mark.parametrize("name", ["gelu", "relu", "silu"])
def test_activations(name):
    g = load_golden("mlp")
    np.testing.assert_allclose(orc.act(g["act_z"], name), g[f"act_{name}"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(orc.act_grad(g["act_z"], name), g[f"actgrad_{name}"], rtol=1e-6, atol=1e-7)


def test_seeded_problem_matches_reference_draws():
    """mlp_problem reproduces bench._mlp_problem's seeded bytes (bench.py:120-130)."""
    g = load_golden("mlp")
    x, w1, w2, idx, p, dy = orc.mlp_problem(256, 64, 128, 8, 2, seed=5)
    np.testing.assert_array_equal(x, g["mlp5_x"])
    np.testing.assert_array_equal(w1, g["mlp5_w1"])
    np.testing.assert_array_equal(w2, g["mlp5_w2"])
    np.testing.assert_array_equal(idx, g["mlp5_idx"])
    np.testing.assert_array_equal(p, g["mlp5_p"])
    np.testing.assert_array_equal(dy, g["mlp5_dy"])


def test_gate_topk_and_backward():
    """gate_forward / topk_select / gate_backward against the reference's outputs."""
    g = load_golden("gate")
    for j in range(int(g["num_gate"])):
        pre = f"g{j}_"
        k, renorm = int(g[pre + "k"]), bool(g[pre + "renorm"])
        gate = orc.gate_probs(g[pre + "x"], g[pre + "wg"])
        np.testing.assert_array_equal(gate, g[pre + "gate"])
        order = np.argsort(-gate, axis=1, kind="stable")[:, :k]
        assert np.array_equal(order, g[pre + "idx"])
        if renorm:
            idx, p = orc.topk_routing(gate, k)
            assert np.array_equal(idx, g[pre + "idx"])
            np.testing.assert_allclose(p, g[pre + "p"], rtol=1e-6, atol=1e-7)
        dz = orc.gate_backward(gate, g[pre + "idx"], g[pre + "grad_p"], renorm)
        np.testing.assert_allclose(dz, g[pre + "dz"], rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(orc.softmax_rows(g[pre + "logits"]), g[pre + "soft"], rtol=1e-6, atol=1e-8)
    tie = g["tie_gate"]
    assert np.array_equal(np.argsort(-tie, axis=1, kind="stable")[:, :3], g["tie_idx"])
