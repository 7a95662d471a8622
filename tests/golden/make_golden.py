"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports scattermlp from /root/reference/pkg/src, runs it on small seeded
problems and writes tests/golden/*.npz.  The fixtures pin the CPU oracle
(oracle/scattermlp_oracle.py) and are also GPU parity targets; nothing at
test or bench time reads /root/reference.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import scattermlp as sm  # noqa: E402
from scattermlp import kernels as sk  # noqa: E402
from scattermlp.core_tensor import ExpertTensor, Matrix  # noqa: E402
from scattermlp.oracle import naive_smoe_mlp  # noqa: E402


def routing_case(rng, t, k, e, flavor):
    """Same three flavours as the reference's conftest.py:12-27."""
    if flavor == "all_to_one":
        idx = np.tile(np.arange(k, dtype=np.int64), (t, 1))
    elif flavor == "skip_one" and e > k:
        idx = np.stack([rng.permutation(e - 1)[:k] for _ in range(t)]).astype(np.int64)
    else:
        logits = Matrix(rng.standard_normal((t, e)).astype(np.float32))
        return sm.topk_select(sm.softmax_rows(logits), k)
    p = rng.random((t, k)).astype(np.float32) + 0.1
    return sm.assignment_routing(idx, e, p)


def routing_fixtures():
    """KATs + stable-order properties of compute_grouped_order (router.py:154-164)."""
    out = {}
    kats = [
        (np.array([[1], [0], [1]]), 2),       # test_router.py:58-63
        (np.array([[0, 2], [1, 0]]), 3),      # test_router.py:66-70
        (np.array([[0, 1], [2, 0]]), 3),      # test_router.py:73-77
        (np.array([[0, 1], [1, 0]]), 2),
    ]
    for i, (idx, e) in enumerate(kats):
        r = sm.assignment_routing(idx, e)
        g = sm.compute_grouped_order(r)
        out[f"kat{i}_idx"] = idx.astype(np.int64)
        out[f"kat{i}_E"] = np.int64(e)
        out[f"kat{i}_o"] = g.o
        out[f"kat{i}_off"] = g.bin_offsets
    rng = np.random.default_rng(1234)
    j = 0
    for flavor in ("gate", "all_to_one", "skip_one"):
        for t, k, e in [(17, 2, 5), (1, 1, 1), (40, 3, 4), (9, 4, 4), (300, 2, 8), (257, 8, 64)]:
            if flavor == "skip_one" and e <= k:
                continue
            r = routing_case(rng, t, k, e, flavor)
            g = sm.compute_grouped_order(r, num_experts=e)
            out[f"case{j}_idx"] = r.expert_idx
            out[f"case{j}_E"] = np.int64(e)
            out[f"case{j}_o"] = g.o
            out[f"case{j}_off"] = g.bin_offsets
            j += 1
    out["num_cases"] = np.int64(j)
    out["num_kats"] = np.int64(len(kats))
    np.savez_compressed(HERE / "routing.npz", **out)


LAYOUTS = {
    "s2g": sk.SCATTERED_TO_GROUPED,
    "g2s": sk.GROUPED_TO_SCATTERED,
    "s2s": sk.SCATTERED_TO_SCATTERED,
    "g2g": sk.GROUPED_TO_GROUPED,
}


def kernel_fixtures():
    """scatter2scatter x 4 layouts x transpose, group, group_xty, scatter_combine."""
    out = {}
    rng = np.random.default_rng(7)
    j = 0
    for lname, layout in LAYOUTS.items():
        for transpose in (False, True):
            for flavor in ("gate", "all_to_one", "skip_one"):
                t, k, e = int(rng.integers(5, 40)), int(rng.integers(1, 4)), int(rng.integers(4, 8))
                d_in, d_out = int(rng.integers(8, 40)), int(rng.integers(8, 40))
                r = routing_case(rng, t, k, e, flavor)
                g = sm.compute_grouped_order(r, num_experts=e)
                rows = t * k if layout.grouped_in else t
                fan_out = 1 if layout.grouped_in else k
                x = rng.uniform(-1, 1, (rows, d_in)).astype(np.float32)
                shape = (e, d_out, d_in) if transpose else (e, d_in, d_out)
                w = (rng.uniform(-1, 1, shape) / np.sqrt(d_in)).astype(np.float32)
                y = sm.scatter2scatter(Matrix(x), ExpertTensor(w), g, fan_out, layout, transpose_w=transpose)
                pre = f"s2s{j}_"
                out.update({pre + "layout": np.array(lname), pre + "transpose": np.int64(transpose),
                            pre + "fan_out": np.int64(fan_out), pre + "idx": r.expert_idx, pre + "E": np.int64(e),
                            pre + "x": x, pre + "w": w, pre + "y": y.data})
                j += 1
    out["num_s2s"] = np.int64(j)
    # group / group_xty / scatter_combine
    r = routing_case(rng, 23, 2, 5, "gate")
    g = sm.compute_grouped_order(r, num_experts=5)
    x = rng.uniform(-1, 1, (23, 12)).astype(np.float32)
    out["grp_idx"] = r.expert_idx
    out["grp_x"] = x
    out["grp_p"] = r.p
    out["grp_plain"] = sm.group(Matrix(x), g, fan_out=2).data
    out["grp_weighted"] = sm.group(Matrix(x), g, weights=r.p_flat, fan_out=2).data
    xg = rng.uniform(-1, 1, (46, 10)).astype(np.float32)
    yg = rng.uniform(-1, 1, (46, 14)).astype(np.float32)
    r2 = routing_case(rng, 23, 2, 6, "skip_one")
    g2 = sm.compute_grouped_order(r2, num_experts=6)
    out["xty_idx"] = r2.expert_idx
    out["xty_x"] = xg
    out["xty_y"] = yg
    out["xty_dw"] = sm.group_xty(Matrix(xg), Matrix(yg), g2).data
    w = (rng.uniform(-1, 1, (5, 12, 9)) / np.sqrt(12)).astype(np.float32)
    out["sc_w"] = w
    out["sc_y"] = sm.scatter_combine(Matrix(x), ExpertTensor(w), g, 2, r.p_flat, 2, False).data
    np.savez_compressed(HERE / "kernels.npz", **out)


def mlp_fixtures():
    """SMoE MLP forward + backward (moe_layers.py:140-211) on seeded problems."""
    out = {}
    cases = [  # (T, d_model, d_expert, E, k, activation, flavor)
        (64, 32, 48, 4, 2, "gelu", "bench"),
        (50, 16, 24, 8, 1, "relu", "bench"),
        (33, 24, 40, 6, 3, "silu", "bench"),
        (40, 16, 32, 4, 2, "gelu", "all_to_one"),
        (40, 16, 32, 5, 2, "gelu", "skip_one"),
        (256, 64, 128, 8, 2, "gelu", "bench"),
    ]
    rng = np.random.default_rng(99)
    for j, (t, d, de, e, k, act, flavor) in enumerate(cases):
        cfg = sm.SmoeMlpConfig(d_model=d, d_expert=de, num_experts=e, k=k, activation=act)
        x = sm.seeded_random_matrix(t, d, j, scale=1.0)
        w1, w2 = sm.init_smoe_mlp_weights(cfg, j + 101)
        if flavor == "bench":
            wg = sm.seeded_random_matrix(d, e, j + 7, scale=1.0 / math.sqrt(d))
            routing = sm.topk_select(sm.gate_forward(x, wg), k)
        else:
            routing = routing_case(rng, t, k, e, flavor)
        order = sm.compute_grouped_order(routing, num_experts=e)
        y, ctx = sm.smoe_mlp_forward(x, w1, w2, routing, order, activation=act, training=True)
        y_naive = naive_smoe_mlp(x, w1, w2, routing, act)
        dy = sm.seeded_random_matrix(t, d, j + 13, scale=1.0)
        grads = sm.smoe_mlp_backward(ctx, dy)
        pre = f"mlp{j}_"
        out.update({
            pre + "act": np.array(act), pre + "E": np.int64(e), pre + "x": x.data, pre + "w1": w1.data,
            pre + "w2": w2.data, pre + "idx": routing.expert_idx, pre + "p": routing.p, pre + "y": y.data,
            pre + "y_naive": y_naive.data, pre + "dy": dy.data, pre + "dx": grads.dx.data,
            pre + "dw1": grads.dw1.data, pre + "dw2": grads.dw2.data, pre + "dp": grads.dp,
        })
    out["num_mlp"] = np.int64(len(cases))
    # activation known values (test_moe_layers.py:56-62 style) over a grid
    z = np.linspace(-6, 6, 97).astype(np.float32)
    for a in ("gelu", "relu", "silu"):
        out[f"act_{a}"] = sm.apply_activation(z, a)
        out[f"actgrad_{a}"] = sm.activation_grad(z, a)
    out["act_z"] = z
    np.savez_compressed(HERE / "mlp.npz", **out)


def parallel_linear_fixtures():
    """ParallelLinear forward/backward with and without p, grouped and scattered X."""
    out = {}
    rng = np.random.default_rng(5)
    j = 0
    for p_given in (False, True):
        for lname in ("s2s", "g2s", "s2g", "g2g"):
            layout = LAYOUTS[lname]
            if p_given and layout.grouped_out:
                continue
            t, k, e, d_in, d_out = 21, 2, 5, 12, 10
            r = routing_case(rng, t, k, e, "gate")
            g = sm.compute_grouped_order(r, num_experts=e)
            rows = t * k if layout.grouped_in else t
            fan_out = 1 if layout.grouped_in else k
            x = rng.uniform(-1, 1, (rows, d_in)).astype(np.float32)
            w = (rng.uniform(-1, 1, (e, d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)
            p = r.p if p_given else None
            y, ctx = sm.parallel_linear_forward(Matrix(x), ExpertTensor(w), g, p=p, fan_out=fan_out,
                                                layout=layout)
            dy = rng.uniform(-1, 1, y.data.shape).astype(np.float32)
            gr = sm.parallel_linear_backward(ctx, Matrix(dy))
            pre = f"pl{j}_"
            out.update({pre + "layout": np.array(lname), pre + "p_given": np.int64(p_given),
                        pre + "fan_out": np.int64(fan_out), pre + "idx": r.expert_idx, pre + "p": r.p,
                        pre + "E": np.int64(e), pre + "x": x, pre + "w": w, pre + "y": y.data, pre + "dy": dy,
                        pre + "dx": gr.dx.data, pre + "dw": gr.dw.data,
                        pre + "dp": gr.dp if gr.dp is not None else np.zeros(0, np.float32)})
            j += 1
    out["num_pl"] = np.int64(j)
    np.savez_compressed(HERE / "parallel_linear.npz", **out)


def momha_fixtures():
    """Routed attention projections (moe_layers.py:406-482), small case."""
    cfg = sm.MomhaConfig(d_model=16, d_head=4, num_heads=4, heads_per_expert=2, num_experts=3, k=2)
    seq_len, b = 8, 2
    x = sm.seeded_random_matrix(b * seq_len, cfg.d_model, 3, scale=1.0)
    wts = sm.init_momha_weights(cfg, 11)
    rng = np.random.default_rng(3)
    r = routing_case(rng, b * seq_len, cfg.k, cfg.num_experts, "gate")
    g = sm.compute_grouped_order(r, num_experts=cfg.num_experts)
    y, ctx = sm.momha_forward(x, wts, r, g, cfg, seq_len)
    dy = sm.seeded_random_matrix(b * seq_len, cfg.d_model, 4, scale=1.0)
    gr = sm.momha_backward(ctx, dy)
    np.savez_compressed(HERE / "momha.npz", x=x.data, wq=wts.wq.data, wk=wts.wk.data, wv=wts.wv.data,
                        wo=wts.wo.data, idx=r.expert_idx, p=r.p, y=y.data, dy=dy.data, dx=gr.dx.data,
                        dwq=gr.dwq.data, dwk=gr.dwk.data, dwv=gr.dwv.data, dwo=gr.dwo.data, dp=gr.dp,
                        seq_len=np.int64(seq_len))


def gate_fixtures():
    """gate_forward / softmax_rows / topk_select / gate_backward (router.py:119-188)."""
    out = {}
    rng = np.random.default_rng(11)
    j = 0
    for t, d, e, k, renorm in [(37, 16, 8, 2, True), (64, 32, 64, 8, True), (20, 8, 5, 3, False), (9, 4, 40, 4, True)]:
        x = Matrix(rng.uniform(-1, 1, (t, d)).astype(np.float32))
        wg = Matrix((rng.uniform(-1, 1, (d, e)) / np.sqrt(d)).astype(np.float32))
        gate = sm.gate_forward(x, wg)
        r = sm.topk_select(gate, k, renormalize=renorm)
        gp = rng.uniform(-1, 1, (t, k)).astype(np.float32)
        dz = sm.gate_backward(r, gp)
        logits = rng.standard_normal((t, e)).astype(np.float32)
        sr = sm.softmax_rows(Matrix(logits))
        r2 = sm.topk_select(sr, k, renormalize=renorm)
        pre = f"g{j}_"
        out.update({pre + "x": x.data, pre + "wg": wg.data, pre + "gate": gate.data, pre + "idx": r.expert_idx,
                    pre + "p": r.p, pre + "k": np.int64(k), pre + "renorm": np.int64(renorm), pre + "grad_p": gp,
                    pre + "dz": dz.data, pre + "logits": logits, pre + "soft": sr.data, pre + "idx2": r2.expert_idx,
                    pre + "p2": r2.p})
        j += 1
    # ties: all-equal rows and duplicated maxima
    tie = np.zeros((3, 6), dtype=np.float32)
    tie[1, [2, 4]] = 1.0
    tie[2, :] = [0.5, 0.1, 0.5, 0.1, 0.5, 0.0]
    rt = sm.topk_select(Matrix(tie), 3, renormalize=False)
    out.update({"tie_gate": tie, "tie_idx": rt.expert_idx, "num_gate": np.int64(j)})
    np.savez_compressed(HERE / "gate.npz", **out)


if __name__ == "__main__":
    gate_fixtures()
    routing_fixtures()
    kernel_fixtures()
    mlp_fixtures()
    parallel_linear_fixtures()
    momha_fixtures()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
