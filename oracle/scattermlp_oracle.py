"""CPU oracle: a NumPy restatement of the reference's ParallelLinear path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs use it, and only as the checker (or as the timed CPU
baseline), never as the thing measured or shipped.

What it restates (each function cites the reference file:line it follows;
paths are relative to /root/reference/pkg/src/scattermlp/):
  * storage is float32, every reduction accumulates in float64 and rounds
    once on write (core_tensor.py:1-10);
  * routing order = stable argsort of the flattened ids + bincount + cumsum;
  * the four scatter2scatter layouts, scatter_combine, group, group_xty,
    the weighted combine and its dp, ParallelLinear forward / backward with
    the buffer-reuse order, and the SMoE MLP forward / backward;
  * the mixture-of-attention layer: slot-query attention and its backward,
    momha_forward / momha_backward (moe_layers.py:270-482).

Parity pinning: tests/golden/*.npz hold input/output vectors produced by
importing the reference itself (tests/golden/make_golden.py, run in the
build container where /root/reference exists); tests/test_oracle_golden.py
checks this restatement against them on every CPU test run.  The reference's
own known-answer vectors (test_router.py:58-77) are asserted
there too.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

F32 = np.float32
F64 = np.float64

# ---------------------------------------------------------------------------
# routing (router.py:154-164, :112-116)


def compute_grouped_order(expert_idx: np.ndarray, num_experts: int):
    """(o, bin_offsets): stable grouping of the T*k slots by expert id (router.py:154-164)."""
    flat = np.asarray(expert_idx, dtype=np.int64).reshape(-1)
    o = np.argsort(flat, kind="stable").astype(np.int64)
    counts = np.bincount(flat, minlength=num_experts).astype(np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return o, offsets


def inverse(o: np.ndarray) -> np.ndarray:
    """scattered slot -> grouped position (router.py:112-116)."""
    inv = np.empty_like(o)
    inv[o] = np.arange(o.size, dtype=o.dtype)
    return inv


def topk_routing(gate: np.ndarray, k: int):
    """Stable top-k with renormalisation in float64 (router.py:137-151)."""
    order = np.argsort(-gate, axis=1, kind="stable")
    idx = order[:, :k].astype(np.int64)
    sel = np.take_along_axis(gate, idx, axis=1)
    p = (sel.astype(F64) / sel.sum(axis=1, keepdims=True, dtype=F64)).astype(gate.dtype)
    return idx, p


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    """Row softmax in float64, stored in the input dtype (router.py:126-134)."""
    z = logits.astype(F64)
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return (e / e.sum(axis=1, keepdims=True)).astype(logits.dtype)


def gate_backward(gate, idx, grad_p, renormalized=True):
    """d logits from d p through renormalisation, selection and softmax (router.py:167-188)."""
    g = gate.astype(F64)
    dp = grad_p.astype(F64)
    gsel = np.take_along_axis(g, idx, axis=1)
    if renormalized:
        s = gsel.sum(axis=1, keepdims=True)
        dgsel = (dp - (dp * (gsel / s)).sum(axis=1, keepdims=True)) / s
    else:
        dgsel = dp
    dg = np.zeros_like(g)
    np.put_along_axis(dg, idx, dgsel, axis=1)
    return (g * (dg - (dg * g).sum(axis=1, keepdims=True))).astype(gate.dtype)


def gate_probs(x: np.ndarray, w_g: np.ndarray) -> np.ndarray:
    """softmax(x @ w_g) in float64, stored float32 (router.py:119-134)."""
    z = x.astype(F64) @ w_g.astype(F64)
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return (e / e.sum(axis=1, keepdims=True)).astype(x.dtype)


# ---------------------------------------------------------------------------
# kernels (kernels.py)


def _bins(offsets):
    for e in range(len(offsets) - 1):
        yield e, int(offsets[e]), int(offsets[e + 1])


def scatter2scatter(x, w, o, offsets, fan_out, grouped_in, grouped_out, transpose_w=False):
    """out[dst(i)] = x[src(i)] @ W[e(i)] per bin, f64 accumulate (kernels.py:143-220)."""
    n = o.size
    d_out = w.shape[1] if transpose_w else w.shape[2]
    out = np.zeros((n, d_out), dtype=x.dtype)
    for e, a, b in _bins(offsets):
        if a == b:
            continue
        rows = np.arange(a, b) if grouped_in else o[a:b] // fan_out
        blk = w[e].T if transpose_w else w[e]
        res = (x[rows].astype(F64) @ blk.astype(F64)).astype(x.dtype)
        if grouped_out:
            out[a:b] = res
        else:
            out[o[a:b]] = res
    return out


def scatter_combine(x, w, o, offsets, fan_out, p_flat, combine_cols, grouped_in):
    """Inference combine fused into the write, f64 accumulate (kernels.py:242-286)."""
    n = o.size
    acc = np.zeros((n // combine_cols, w.shape[2]), dtype=F64)
    for e, a, b in _bins(offsets):
        if a == b:
            continue
        rows = np.arange(a, b) if grouped_in else o[a:b] // fan_out
        blk = x[rows].astype(F64) @ w[e].astype(F64)
        slots = o[a:b]
        blk *= p_flat[slots].astype(F64)[:, None]
        np.add.at(acc, slots // combine_cols, blk)
    return acc.astype(x.dtype)


def group(x, o, weights=None, fan_out=1):
    """row i <- x[o[i] // fan_out] * weights[o[i]] (kernels.py:289-326)."""
    out = x[o // fan_out].copy()
    if weights is not None:
        out *= weights[o][:, None].astype(x.dtype)
    return out


def group_xty(xg, yg, offsets):
    """dW[e] = xg[bin]^T @ yg[bin] in f64; empty bin -> zeros (kernels.py:329-361)."""
    e_count = len(offsets) - 1
    dw = np.zeros((e_count, xg.shape[1], yg.shape[1]), dtype=xg.dtype)
    for e, a, b in _bins(offsets):
        if a < b:
            dw[e] = (xg[a:b].astype(F64).T @ yg[a:b].astype(F64)).astype(xg.dtype)
    return dw


def combine(p, y_hat):
    """Y[s] = sum_j p[s,j] Y_hat[s*J+j] in f64 (parallel_linear.py:69-73)."""
    s, j = p.shape
    v = y_hat.reshape(s, j, y_hat.shape[1]).astype(F64)
    return np.einsum("sj,sjd->sd", p.astype(F64), v).astype(y_hat.dtype)


def combine_grad_p(dy, y_hat, s, j):
    """dp[s,j] = <dY[s], Y_hat[s*J+j]> in f64 (parallel_linear.py:198-206)."""
    v = y_hat.reshape(s, j, y_hat.shape[1]).astype(F64)
    return np.einsum("sd,sjd->sj", dy.astype(F64), v).astype(F32)


def fanout_reduce(g, fan_out):
    """dX[t] = sum_j G[t*F + j] in f64 (parallel_linear.py:259-266)."""
    t = g.shape[0] // fan_out
    return g.reshape(t, fan_out, g.shape[1]).sum(axis=1, dtype=F64).astype(g.dtype)


# ---------------------------------------------------------------------------
# activations (moe_layers.py:42-90), f64 math rounded once

_INV_SQRT2 = 1.0 / math.sqrt(2.0)
_INV_SQRT_2PI = 1.0 / math.sqrt(2.0 * math.pi)


def act(z, name):
    z64 = z.astype(F64)
    if name == "gelu":
        r = 0.5 * z64 * (1.0 + erf(z64 * _INV_SQRT2))
    elif name == "relu":
        r = np.maximum(z64, 0.0)
    elif name == "silu":
        r = z64 / (1.0 + np.exp(-z64))
    else:
        raise ValueError(name)
    return r.astype(z.dtype)


def act_grad(z, name):
    z64 = z.astype(F64)
    if name == "gelu":
        r = 0.5 * (1.0 + erf(z64 * _INV_SQRT2)) + z64 * np.exp(-0.5 * z64 * z64) * _INV_SQRT_2PI
    elif name == "relu":
        r = (z64 > 0.0).astype(F64)
    elif name == "silu":
        s = 1.0 / (1.0 + np.exp(-z64))
        r = s * (1.0 + z64 * (1.0 - s))
    else:
        raise ValueError(name)
    return r.astype(z.dtype)


# ---------------------------------------------------------------------------
# ParallelLinear (parallel_linear.py:85-269) and the SMoE MLP (moe_layers.py:140-211)


def pl_forward(x, w, o, offsets, p, fan_out, grouped_in, grouped_out):
    """(y, y_hat): Alg. 1 in training mode (parallel_linear.py:85-141)."""
    if p is None:
        y_hat = scatter2scatter(x, w, o, offsets, fan_out, grouped_in, grouped_out)
        return y_hat, y_hat
    y_hat = scatter2scatter(x, w, o, offsets, fan_out, grouped_in, False)
    return combine(p, y_hat), y_hat


def pl_backward(x, w, o, offsets, p, fan_out, x_grouped, y_grouped, y_hat, dy):
    """(dx, dw, dp): Alg. 2 (parallel_linear.py:157-269)."""
    dp = None
    if p is not None:
        s, j = p.shape
        dp = combine_grad_p(dy, y_hat, s, j)
        gdy = group(dy, o, weights=p.reshape(-1), fan_out=j)
    elif y_grouped:
        gdy = dy
    else:
        gdy = group(dy, o, fan_out=1)
    xbar = x if x_grouped else group(x, o, fan_out=fan_out)
    dw = group_xty(xbar, gdy, offsets)
    if x_grouped:
        dx = scatter2scatter(gdy, w, o, offsets, 1, True, True, transpose_w=True)
    else:
        g = scatter2scatter(gdy, w, o, offsets, 1, True, False, transpose_w=True)
        dx = g if fan_out == 1 else fanout_reduce(g, fan_out)
    return dx, dw, dp


def smoe_mlp_forward(x, w1, w2, expert_idx, p, num_experts, activation="gelu"):
    """Returns y and the saved state (moe_layers.py:140-182)."""
    k = expert_idx.shape[1]
    o, off = compute_grouped_order(expert_idx, num_experts)
    h_pre = scatter2scatter(x, w1, o, off, k, False, True)
    h = act(h_pre, activation)
    y_hat = scatter2scatter(h, w2, o, off, 1, True, False)
    y = combine(p, y_hat)
    return y, dict(o=o, off=off, h_pre=h_pre, h=h, y_hat=y_hat, k=k)


def smoe_mlp_backward(x, w1, w2, p, state, dy, activation="gelu"):
    """(dx, dw1, dw2, dp) (moe_layers.py:185-211)."""
    o, off, k = state["o"], state["off"], state["k"]
    dh, dw2, dp = pl_backward(state["h"], w2, o, off, p, 1, True, False, state["y_hat"], dy)
    dh = (dh * act_grad(state["h_pre"], activation)).astype(x.dtype)
    dx, dw1, _ = pl_backward(x, w1, o, off, None, k, False, True, None, dh)
    return dx, dw1, dw2, dp


def naive_smoe_mlp(x, w1, w2, expert_idx, p, activation="gelu"):
    """Per-token, per-selection evaluation that never consults the order (oracle.py:74-95)."""
    t, k = expert_idx.shape
    y = np.zeros((t, w2.shape[2]), dtype=F64)
    for tok in range(t):
        xt = x[tok].astype(F64)
        for sel in range(k):
            e = int(expert_idx[tok, sel])
            h = act(xt @ w1[e].astype(F64), activation).astype(F64)
            y[tok] += float(p[tok, sel]) * (h @ w2[e].astype(F64))
    return y.astype(x.dtype)


# ---------------------------------------------------------------------------
# Mixture of multi-head attention (moe_layers.py:270-482)


def _causal_chunks(n_tokens, seq_len, k, chunk_slots=2048):
    """(token lo, token hi, slot lo, slot hi) query chunks, never crossing a sequence."""
    if n_tokens % seq_len:
        raise ValueError(f"token count {n_tokens} is not divisible by seq_len {seq_len}")
    for lo in range(0, n_tokens, seq_len):
        for s0 in range(lo * k, (lo + seq_len) * k, chunk_slots):
            yield lo, lo + seq_len, s0, min(s0 + chunk_slots, (lo + seq_len) * k)


def attention(q, keys, values, k, seq_len, d_head, causal=True):
    """Per-slot queries vs dense keys (moe_layers.py:280-327).

    Slots are chronological (slot s belongs to token s // k, as momha_forward
    lays them out, :441); query head columns [c0, c0 + d_head) attend with the
    same columns of the keys / values of the slot's sequence, causally.  Scores
    and softmax in f64, one rounding.  Query rows are processed in chunks so a
    4096-token sequence stays within a few hundred MB.
    """
    n = keys.shape[0]
    out = np.empty(q.shape, dtype=q.dtype)
    scale = 1.0 / math.sqrt(d_head)
    qd, kd, vd = q.astype(F64), keys.astype(F64), values.astype(F64)
    for lo, hi, s0, s1 in _causal_chunks(n, seq_len, k):
        times = np.arange(s0, s1) // k - lo
        mask = times[:, None] < np.arange(hi - lo)[None, :] if causal else None
        for c0 in range(0, q.shape[1], d_head):
            c = slice(c0, c0 + d_head)
            sc = (qd[s0:s1, c] @ kd[lo:hi, c].T) * scale
            if mask is not None:
                sc = np.where(mask, -np.inf, sc)
            sc -= sc.max(axis=1, keepdims=True)
            wts = np.exp(sc)
            wts /= wts.sum(axis=1, keepdims=True)
            out[s0:s1, c] = (wts @ vd[lo:hi, c]).astype(q.dtype)
    return out


def attention_backward(q, keys, values, k, seq_len, d_head, causal, d_out):
    """(dq, dkeys, dvalues) with recomputed probabilities (moe_layers.py:330-377)."""
    n = keys.shape[0]
    scale = 1.0 / math.sqrt(d_head)
    qd, kd, vd, god = q.astype(F64), keys.astype(F64), values.astype(F64), d_out.astype(F64)
    dq = np.zeros_like(qd)
    dk = np.zeros_like(kd)
    dv = np.zeros_like(vd)
    for lo, hi, s0, s1 in _causal_chunks(n, seq_len, k):
        times = np.arange(s0, s1) // k - lo
        mask = times[:, None] < np.arange(hi - lo)[None, :] if causal else None
        for c0 in range(0, q.shape[1], d_head):
            c = slice(c0, c0 + d_head)
            sc = (qd[s0:s1, c] @ kd[lo:hi, c].T) * scale
            if mask is not None:
                sc = np.where(mask, -np.inf, sc)
            sc -= sc.max(axis=1, keepdims=True)
            pr = np.exp(sc)
            pr /= pr.sum(axis=1, keepdims=True)
            g = god[s0:s1, c]
            dpr = g @ vd[lo:hi, c].T
            ds = pr * (dpr - (dpr * pr).sum(axis=1, keepdims=True))
            dq[s0:s1, c] = (ds @ kd[lo:hi, c]) * scale
            dk[lo:hi, c] += (ds.T @ qd[s0:s1, c]) * scale
            dv[lo:hi, c] += pr.T @ g
    return dq.astype(q.dtype), dk.astype(q.dtype), dv.astype(q.dtype)


def _matmul(a, b):
    """core_tensor.matmul (core_tensor.py:130-143): f64 accumulation, one rounding."""
    return (a.astype(F64) @ b.astype(F64)).astype(a.dtype)


def momha_forward(x, wq, wk, wv, wo, expert_idx, p, num_experts, seq_len, d_head, causal=True):
    """y and the saved state (moe_layers.py:406-457): dense K/V, routed Q / O projections."""
    k = expert_idx.shape[1]
    o, off = compute_grouped_order(expert_idx, num_experts)
    keys, values = _matmul(x, wk), _matmul(x, wv)
    q = scatter2scatter(x, wq, o, off, k, False, False)
    attn = attention(q, keys, values, k, seq_len, d_head, causal)
    y, y_hat = pl_forward(attn, wo, o, off, p, 1, False, False)
    return y, dict(o=o, off=off, k=k, q=q, keys=keys, values=values, attn=attn, y_hat=y_hat,
                   seq_len=seq_len, d_head=d_head, causal=causal)


def momha_backward(x, wq, wk, wv, wo, p, state, dy):
    """(dx, dwq, dwk, dwv, dwo, dp) (moe_layers.py:460-482)."""
    o, off, k = state["o"], state["off"], state["k"]
    dattn, dwo, dp = pl_backward(state["attn"], wo, o, off, p, 1, False, False, state["y_hat"], dy)
    dq, dk, dv = attention_backward(state["q"], state["keys"], state["values"], k, state["seq_len"],
                                    state["d_head"], state["causal"], dattn)
    dx_q, dwq, _ = pl_backward(x, wq, o, off, None, k, False, False, None, dq)
    x64 = x.astype(F64)
    dwk = (x64.T @ dk.astype(F64)).astype(x.dtype)
    dwv = (x64.T @ dv.astype(F64)).astype(x.dtype)
    dx_kv = dk.astype(F64) @ wk.astype(F64).T + dv.astype(F64) @ wv.astype(F64).T
    dx = (dx_q.astype(F64) + dx_kv).astype(x.dtype)
    return dx, dwq, dwk, dwv, dwo, dp


# ---------------------------------------------------------------------------
# seeded problem construction (bench.py:120-130, moe_layers.py:111-121, core_tensor.py:146-168)


def seeded_uniform(shape, seed, scale=1.0):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-scale, scale, size=shape).astype(F32)


def mlp_problem(t, d_model, d_expert, num_experts, k, seed=0):
    """Seeded X, W1, W2, routing and dY, as bench._mlp_problem draws them."""
    x = seeded_uniform((t, d_model), seed)
    w1 = seeded_uniform((num_experts, d_model, d_expert), seed + 101, 1.0 / math.sqrt(d_model))
    w2 = seeded_uniform((num_experts, d_expert, d_model), seed + 102, 1.0 / math.sqrt(d_expert))
    wg = seeded_uniform((d_model, num_experts), seed + 7, 1.0 / math.sqrt(d_model))
    idx, p = topk_routing(gate_probs(x, wg), k)
    dy = seeded_uniform((t, d_model), seed + 13)
    return x, w1, w2, idx, p, dy
