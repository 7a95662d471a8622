"""Routed layers built from the expert-linear transform (GPU).

Mirrors the reference moe_layers.py (/root/reference/pkg/src/scattermlp/moe_layers.py):
activations (:42-90), SmoeMlpConfig / init_smoe_mlp_weights (:93-121),
smoe_mlp_forward / smoe_mlp_backward (:140-211), MomhaConfig / MomhaWeights /
init_momha_weights (:214-267), attention / attention_backward (:280-377),
momha_forward / momha_backward (:406-482).

B200 changes (same results, fewer passes over HBM):
  * the activation is fused into the first transform's epilogue, which writes
    the retained pre-activation and the activated hidden state in one pass
    (reference: copy + in-place activation, :169-175);
  * the activation derivative is fused into the output transform's
    input-gradient kernel (reference: a separate multiply, :205-206).
The buffer-reuse discipline of smoe_mlp_backward (:198-211) is kept exactly.

The attention core of MoMHA (between the two routed projections) is outside
the ParallelLinear hot path: it runs as torch's fused
scaled-dot-product attention (library flash / cuDNN kernels) in grouped-query
form, and the shared K/V projections as library GEMMs.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from . import parallel_linear as pl
from .errors import require_dims
from .kernels import (
    GROUPED_TO_GROUPED,
    GROUPED_TO_SCATTERED,
    SCATTERED_TO_GROUPED,
    SCATTERED_TO_SCATTERED,
    LayoutFlag,
    TileConfig,
)
from .router import GroupedOrder, RoutingResult

ACTIVATIONS = ("gelu", "relu", "silu")


def _activation(name: str) -> str:
    if name not in ACTIVATIONS:
        raise ValueError(f"unknown activation {name!r}; choose from {sorted(ACTIVATIONS)}")
    return name


def apply_activation(values: torch.Tensor, name: str) -> torch.Tensor:
    """Elementwise activation (fp32 math, rounded once), moe_layers.py:75-78."""
    return K.activation_kernel(values, _activation(name), derivative=False)


def activation_grad(pre: torch.Tensor, name: str) -> torch.Tensor:
    """Elementwise activation derivative, moe_layers.py:81-83."""
    return K.activation_kernel(pre, _activation(name), derivative=True)


@dataclass(frozen=True)
class SmoeMlpConfig:
    """Shapes for the routed MLP: two expert stacks around one activation (moe_layers.py:93-108)."""

    d_model: int
    d_expert: int
    num_experts: int
    k: int
    activation: str = "gelu"

    def __post_init__(self):
        if min(self.d_model, self.d_expert, self.num_experts, self.k) < 1:
            raise ValueError(f"all MLP dimensions must be >= 1: {self}")
        if self.k > self.num_experts:
            raise ValueError(f"k={self.k} exceeds expert count {self.num_experts}")
        _activation(self.activation)


def seeded_expert_tensor(num_experts, d_in, d_out, seed, scale=1.0, dtype=torch.float32,
                         device="cuda") -> torch.Tensor:
    """U[-scale, scale] from PCG64(seed), the reference's draw (core_tensor.py:155-168)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    arr = rng.uniform(-scale, scale, size=(num_experts, d_in, d_out)).astype(np.float32)
    return torch.from_numpy(arr).to(device=device, dtype=dtype)


def seeded_matrix(rows, cols, seed, scale=1.0, dtype=torch.float32, device="cuda") -> torch.Tensor:
    """U[-scale, scale] from PCG64(seed) (core_tensor.py:146-152)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    arr = rng.uniform(-scale, scale, size=(rows, cols)).astype(np.float32)
    return torch.from_numpy(arr).to(device=device, dtype=dtype)


def init_smoe_mlp_weights(config: SmoeMlpConfig, seed: int, dtype=torch.float32, device="cuda",
                          source: str = "pcg64"):
    """Seeded (W1, W2) expert stacks with 1/sqrt(d_in) scaling (moe_layers.py:111-121).

    source="pcg64" reproduces the reference's bytes exactly (CPU draw, upload);
    source="device" draws U[-s, s] with torch on the GPU (perf-only runs).
    """
    e, d, de = config.num_experts, config.d_model, config.d_expert
    s1, s2 = 1.0 / math.sqrt(d), 1.0 / math.sqrt(de)
    if source == "pcg64":
        return (seeded_expert_tensor(e, d, de, seed, s1, dtype, device),
                seeded_expert_tensor(e, de, d, seed + 1, s2, dtype, device))
    g = torch.Generator(device=device).manual_seed(seed)
    w1 = (torch.rand((e, d, de), generator=g, device=device, dtype=torch.float32) * 2 - 1).mul_(s1).to(dtype)
    w2 = (torch.rand((e, de, d), generator=g, device=device, dtype=torch.float32) * 2 - 1).mul_(s2).to(dtype)
    return w1, w2


@dataclass
class _ScaledState:
    """Saved tensors of the routing-weight-scaled MLP path (see smoe_mlp_forward)."""
    x: torch.Tensor
    w1: torch.Tensor
    w2: torch.Tensor
    order: GroupedOrder
    p: torch.Tensor
    hp: torch.Tensor        # p[slot] * act(h_pre), grouped (the layer-2 input)
    y_hat_p: torch.Tensor   # layer-2 output rows p * Y_hat in slot order (storage reused in the backward)


@dataclass
class SmoeMlpContext:
    hidden_ctx: pl.LinearContext | None
    output_ctx: pl.LinearContext | None
    h_pre: torch.Tensor
    activation: str
    scaled: _ScaledState | None = None


# The routing weight moves through layer 2: layer 1's epilogue writes
# p * act(h_pre), so Y = sum over the k slot rows of layer 2's output (an
# unweighted reduce), and dp comes out of the dH GEMM's epilogue as
# <dY W2^T, act(h_pre)> = <dY, Y_hat> — no retained Y_hat and no dp pass over
# it.  SMOE_MLP_SCALED=0 runs the reference's literal sequence instead
# (moe_layers.py:140-211: combine after layer 2, dp from the retained output).
_SCALED = os.environ.get("SMOE_MLP_SCALED", "1") != "0"


# SMOE_GROUPED_REDUCE=1: the k-summed GEMMs (layer 2, the input gradient) write
# grouped rows (TMA slab stores) and the k-sum reads them through the inverse
# permutation.  Measured against scattered-row outputs (alternating, one box):
# C1 906-910 k vs 907-909 k tok/s, C2 1.593-1.598 M vs 1.582-1.600 M — the
# staged scattered-row epilogue is not what limits those GEMMs; off.
_GROUPED_REDUCE = os.environ.get("SMOE_GROUPED_REDUCE", "0") == "1"

# SMOE_L1_GROUPED=1: the scaled forward copies X into grouped order (into the
# layer-2 output's storage, so no extra buffer) and runs layer 1 as a TMA-fed
# grouped-input GEMM instead of gathering X's rows inside the GEMM.  Layer 1
# drops 6.25 -> 5.77 ms (C1) and 3.25 -> 2.94 ms (C2), but under the power cap
# the other GEMMs slow by about as much and the copy is one more pass: C1
# 912-915 k vs 909-914 k tok/s, C2 1.588-1.591 M vs 1.594-1.601 M; off.
_L1_GROUPED = os.environ.get("SMOE_L1_GROUPED", "0") == "1"


def set_scaled(enabled: bool) -> bool:
    """Select the routing-weight-scaled MLP path (True) or the literal one; returns the previous value."""
    global _SCALED
    prev, _SCALED = _SCALED, bool(enabled)
    return prev


def _scaled_ok(x: torch.Tensor, w1: torch.Tensor, order: GroupedOrder) -> bool:
    return (_SCALED and x.dtype == torch.bfloat16 and K.get_engine() != "simt" and order.num_experts <= 128
            and os.environ.get("SMOE_TC_CTAS", "2") != "1" and x.shape[1] % 8 == 0 and w1.shape[2] % 8 == 0)


@dataclass
class SmoeMlpGradients:
    dx: torch.Tensor
    dw1: torch.Tensor
    dw2: torch.Tensor
    dp: torch.Tensor


def smoe_mlp_forward(
    x: torch.Tensor,
    w1: torch.Tensor,
    w2: torch.Tensor,
    routing: RoutingResult,
    order: GroupedOrder,
    *,
    activation: str = "gelu",
    training: bool = True,
    tile: TileConfig | None = None,
    ledger=None,
) -> tuple[torch.Tensor, SmoeMlpContext | None]:
    """Y[t] = sum_i p[t,i] * act(x[t] @ W1[e_i]) @ W2[e_i]  (moe_layers.py:140-182).

    The hidden state exists only in grouped layout (T*k x d_expert).
    """
    require_dims(w1.shape[2] == w2.shape[1], "expert hidden widths", tuple(w1.shape[1:]), tuple(w2.shape[1:]))
    require_dims(w1.shape[1] == x.shape[1], "input width vs W1", tuple(x.shape), tuple(w1.shape[1:]))
    require_dims(w2.shape[2] == x.shape[1], "W2 output width vs model width", tuple(w2.shape[1:]), (x.shape[1],))
    _activation(activation)
    k = routing.k
    if order.num_slots != x.shape[0] * k:
        raise ValueError(f"order covers {order.num_slots} slots but routing implies {x.shape[0]}*{k}")
    n, de = order.num_slots, w1.shape[2]
    if training and _scaled_ok(x, w1, order):
        p_flat = routing.p.reshape(-1).to(torch.float32).contiguous()
        h_pre = torch.empty((n, de), dtype=x.dtype, device=x.device)
        hp = torch.empty((n, de), dtype=x.dtype, device=x.device)
        y_hat_p = torch.empty((n, w2.shape[2]), dtype=x.dtype, device=x.device)
        if _L1_GROUPED and w2.shape[2] == x.shape[1]:
            # grouped X staged in the layer-2 output's storage (dead until layer 2
            # writes it): layer 1 runs TMA-fed instead of gathering rows
            xg = K.group(x, order, fan_out=k, out=y_hat_p)
            K.scatter2scatter_scaled(xg, w1, order, 1, GROUPED_TO_GROUPED, row_scale=p_flat,
                                     activation=activation, out=h_pre, act_out=hp)
        else:
            K.scatter2scatter_scaled(x, w1, order, k, SCATTERED_TO_GROUPED, row_scale=p_flat,
                                     activation=activation, out=h_pre, act_out=hp)
        if _GROUPED_REDUCE:
            # layer 2 writes grouped rows (whole 32-row slabs leave by TMA) and the
            # k-sum gathers each token's rows through the inverse permutation
            K.scatter2scatter(hp, w2, order, 1, GROUPED_TO_GROUPED, out=y_hat_p)
            y = K.fanout_reduce(y_hat_p, k, inverse=order.inverse())
        else:
            K.scatter2scatter(hp, w2, order, 1, GROUPED_TO_SCATTERED, out=y_hat_p)
            y = K.fanout_reduce(y_hat_p, k)
        if ledger:
            ledger.alloc("mlp.hidden.y", n, de, "forward")
            ledger.alloc("mlp.h_preactivation", n, de, "backward")
            ledger.alloc("mlp.output.y_hat", n, w2.shape[2], "backward")
            ledger.alloc("mlp.output.y", y.shape[0], y.shape[1], "forward")
        st = _ScaledState(x=x, w1=w1, w2=w2, order=order, p=routing.p, hp=hp, y_hat_p=y_hat_p)
        return y, SmoeMlpContext(hidden_ctx=None, output_ctx=None, h_pre=h_pre, activation=activation, scaled=st)
    if training:
        h_pre = torch.empty((n, de), dtype=x.dtype, device=x.device)
        h = torch.empty((n, de), dtype=x.dtype, device=x.device)
        K.scatter2scatter(x, w1, order, k, SCATTERED_TO_GROUPED, tile, out=h_pre,
                          activation=activation, act_out=h)
        if ledger:
            ledger.alloc("mlp.hidden.y", n, de, "forward")
            ledger.alloc("mlp.h_preactivation", n, de, "backward")
        hidden_ctx = pl.LinearContext(x=x, w=w1, order=order, p=None, fan_out=k, x_was_grouped=False,
                                      y_was_grouped=True, y_hat=h)
    else:
        h = K.scatter2scatter(x, w1, order, k, SCATTERED_TO_GROUPED, tile, activation=activation)
        if ledger:
            ledger.alloc("mlp.hidden.y", n, de, "forward")
        h_pre = hidden_ctx = None
    y, output_ctx = pl.forward(h, w2, order, p=routing.p, fan_out=1, layout=GROUPED_TO_SCATTERED,
                               tile=tile, training=training, ledger=ledger, name="mlp.output")
    if not training:
        return y, None
    return y, SmoeMlpContext(hidden_ctx=hidden_ctx, output_ctx=output_ctx, h_pre=h_pre, activation=activation)


def smoe_mlp_backward(ctx: SmoeMlpContext, dy: torch.Tensor, *, tile: TileConfig | None = None,
                      ledger=None, on_dx=None) -> SmoeMlpGradients:
    """Gradients for the routed MLP; stops at dp (moe_layers.py:185-211).

    Reuse: the output transform's input gradients land in the activated hidden
    buffer (after dW2 consumed it) with act'(h_pre) fused in; the retained
    pre-combine output's storage takes the hidden transform's grouped input.
    No new T*k-row buffer is allocated.

    on_dx(dx, dp): optional hook, called as soon as the kernels producing dX
    and dp are enqueued on the current stream (the bf16 path enqueues the
    input gradient before the last weight gradient), so a caller can start
    dX's copy or communication while dW1 computes.
    """
    if ctx.scaled is not None:
        return _scaled_backward(ctx, dy, on_dx)
    out_ctx = ctx.output_ctx
    hid_ctx = ctx.hidden_ctx
    out_ctx.scratch_grouped_x = out_ctx.x
    g2 = pl.backward(out_ctx, dy, tile=tile, ledger=ledger, name="mlp.output",
                     dx_activation_grad=(ctx.h_pre, ctx.activation))
    dh = g2.dx
    hid_ctx.scratch_grouped_x = out_ctx.y_hat
    g1 = pl.backward(hid_ctx, dh, tile=tile, ledger=ledger, name="mlp.hidden")
    if on_dx is not None:
        on_dx(g1.dx, g2.dp)
    return SmoeMlpGradients(dx=g1.dx, dw1=g1.dw, dw2=g2.dw, dp=g2.dp)


def _scaled_backward(ctx: SmoeMlpContext, dy: torch.Tensor, on_dx=None) -> SmoeMlpGradients:
    """Backward of the routing-weight-scaled path; the reference's buffer reuse
    (moe_layers.py:198-211): grouped dY lives in the retained output's
    storage, dH overwrites p * act(h_pre) after dW2 consumed it.  The input
    gradient is produced before dW1 (dX is what the upstream layer waits for):
    the slot input-gradients take grouped dY's storage, and after their k-sum
    the grouped input for dW1 reuses it — still no new T*k-row buffer."""
    st = ctx.scaled
    order, k = st.order, st.p.shape[1]
    t = st.p.shape[0]
    if tuple(dy.shape) != (t, st.w2.shape[2]):
        require_dims(False, "dy vs combine output", tuple(dy.shape), (t, st.w2.shape[2]))
    dy = dy.contiguous()
    p_flat = st.p.reshape(-1).to(torch.float32).contiguous()
    de = st.w1.shape[2]
    dyg = K.group(dy, order, fan_out=k, out=st.y_hat_p)
    dw2 = K.group_xty(st.hp, dyg, order)
    parts = torch.empty((order.num_slots, K.dp_parts(de)), dtype=torch.float32, device=dy.device)
    dh = K.scatter2scatter_scaled(dyg, st.w2, order, 1, GROUPED_TO_GROUPED, row_scale=p_flat,
                                  activation=ctx.activation, out=st.hp, act_grad_of=ctx.h_pre,
                                  dp_partials=parts, transpose_w=True)
    dp = K.dp_from_partials(parts, order, t, k)
    if _GROUPED_REDUCE:
        slot = K.scatter2scatter(dh, st.w1, order, 1, GROUPED_TO_GROUPED, transpose_w=True, out=dyg)
        dx = K.fanout_reduce(slot, k, inverse=order.inverse())
    else:
        slot = K.scatter2scatter(dh, st.w1, order, 1, GROUPED_TO_SCATTERED, transpose_w=True, out=dyg)
        dx = K.fanout_reduce(slot, k)
    if on_dx is not None:
        on_dx(dx, dp)
    if pl._gather_ok(de, st.x) and order.num_experts <= 128:
        dw1 = K.group_xty_scattered(st.x, dh, order, x_fan_out=k, y_grouped=True)
    else:
        # stream order: the k-sum above has read the slot gradients first
        xbar = K.group(st.x, order, fan_out=k, out=dyg)
        dw1 = K.group_xty(xbar, dh, order)
    return SmoeMlpGradients(dx=dx, dw1=dw1, dw2=dw2, dp=dp)


class _SmoeMlpFunction(torch.autograd.Function):
    @staticmethod
    def forward(actx, x, w1, w2, p, routing, order, activation):
        y, mctx = smoe_mlp_forward(x.detach(), w1.detach(), w2.detach(), routing, order,
                                   activation=activation, training=True)
        actx.mctx = mctx
        return y

    @staticmethod
    def backward(actx, dy):
        g = smoe_mlp_backward(actx.mctx, dy.contiguous())
        actx.mctx = None
        return g.dx, g.dw1, g.dw2, g.dp, None, None, None


class SmoeMlp(torch.nn.Module):
    """The SMoE MLP module (north_star): two expert stacks around one activation.

    forward(x, routing, order) -> (T, d_model); differentiable wrt x, W1, W2 and p
    (routing.p), through the fused GPU forward/backward above.
    """

    def __init__(self, config: SmoeMlpConfig, dtype=torch.bfloat16, device="cuda", seed: int = 0,
                 source: str = "device"):
        super().__init__()
        self.config = config
        w1, w2 = init_smoe_mlp_weights(config, seed, dtype=dtype, device=device, source=source)
        self.w1 = torch.nn.Parameter(w1)
        self.w2 = torch.nn.Parameter(w2)

    def forward(self, x: torch.Tensor, routing: RoutingResult, order: GroupedOrder) -> torch.Tensor:
        if not self.training and not torch.is_grad_enabled():
            y, _ = smoe_mlp_forward(x, self.w1, self.w2, routing, order, activation=self.config.activation,
                                    training=False)
            return y
        return _SmoeMlpFunction.apply(x, self.w1, self.w2, routing.p, routing, order, self.config.activation)


# ---------------------------------------------------------------------------
# Mixture of multi-head attention (MoMHA): routed query / output projections.

@dataclass(frozen=True)
class MomhaConfig:
    """Routed multi-head attention shapes (moe_layers.py:214-247)."""

    d_model: int
    d_head: int
    num_heads: int
    heads_per_expert: int
    num_experts: int
    k: int
    causal: bool = True

    def __post_init__(self):
        if min(self.d_model, self.d_head, self.num_heads, self.heads_per_expert, self.num_experts, self.k) < 1:
            raise ValueError(f"all attention dimensions must be >= 1: {self}")
        if self.num_heads != self.k * self.heads_per_expert:
            raise ValueError(f"num_heads ({self.num_heads}) must equal k ({self.k}) * "
                             f"heads_per_expert ({self.heads_per_expert})")
        if self.k > self.num_experts:
            raise ValueError(f"k={self.k} exceeds expert count {self.num_experts}")

    @property
    def d_proj(self) -> int:
        return self.heads_per_expert * self.d_head


@dataclass
class MomhaWeights:
    wq: torch.Tensor  # (E, d_model, d_proj)
    wk: torch.Tensor  # (d_model, d_proj), shared
    wv: torch.Tensor  # (d_model, d_proj), shared
    wo: torch.Tensor  # (E, d_proj, d_model)


def init_momha_weights(config: MomhaConfig, seed: int, dtype=torch.float32, device="cuda") -> MomhaWeights:
    """Seeded MoMHA weights, same draws as moe_layers.py:257-267."""
    d, dp_ = config.d_model, config.d_proj
    s_in, s_out = 1.0 / math.sqrt(d), 1.0 / math.sqrt(dp_)
    return MomhaWeights(
        wq=seeded_expert_tensor(config.num_experts, d, dp_, seed, s_in, dtype, device),
        wk=seeded_matrix(d, dp_, seed + 1, s_in, dtype, device),
        wv=seeded_matrix(d, dp_, seed + 2, s_in, dtype, device),
        wo=seeded_expert_tensor(config.num_experts, dp_, d, seed + 3, s_out, dtype, device),
    )


_GQA = os.environ.get("SMOE_MOMHA_GQA", "1") != "0"


# SMOE_MOMHA_GROUPED=0: slot rows in slot order around the attention core (A/B)
_MOMHA_GROUPED = os.environ.get("SMOE_MOMHA_GROUPED", "1") != "0"
# SMOE_MOMHA_HEADS_OUT=0: the q projection and the attention-output gradient
# leave their GEMMs as grouped rows and move to the head layout separately (A/B)
_MOMHA_HEADS_OUT = os.environ.get("SMOE_MOMHA_HEADS_OUT", "1") != "0"


def _contig16(t: torch.Tensor) -> torch.Tensor:
    """Contiguous copy of a permuted view whose last dimension is contiguous, moved
    as 16-byte elements (4x faster than the element-wise bf16 permute copy)."""
    if t.is_contiguous():
        return t
    return t.view(torch.complex128).contiguous().view(t.dtype)


def _attn_core(q, keys, values, seq_len, d_head, k, causal):
    """Slot queries (T*k, d_proj) in chronological order vs dense K/V (T, d_proj).

    Query head (slot, j) attends with K/V head j of its sequence; causal within
    the sequence (moe_layers.py:280-327).  The k slots of a token sit at the
    token's position, so the core is causal attention with k query heads per
    K/V head (grouped-query layout): query head hh*k + j of a token is its slot
    j's head hh.  Runs as one fused scaled-dot-product attention (flash /
    cuDNN kernels for bf16), in the input dtype.
    """
    n = keys.shape[0]
    b = n // seq_len
    h = q.shape[1] // d_head
    qh = q.view(b, seq_len, k, h, d_head).permute(0, 3, 2, 1, 4).reshape(b, h * k, seq_len, d_head)
    kh = keys.view(b, seq_len, h, d_head).transpose(1, 2)
    vh = values.view(b, seq_len, h, d_head).transpose(1, 2)
    if _GQA:
        # K/V head hh serves query heads hh*k .. hh*k+k-1 without materialising k copies
        out = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=causal, enable_gqa=k > 1)
    else:
        out = torch.nn.functional.scaled_dot_product_attention(qh, kh.repeat_interleave(k, dim=1),
                                                               vh.repeat_interleave(k, dim=1), is_causal=causal)
    return out.view(b, h, k, seq_len, d_head).permute(0, 3, 2, 1, 4).reshape(b * seq_len * k, h * d_head)


def _mm(a, b):
    """Dense projection: bf16 on the tensor cores with fp32 accumulation, fp32 exact-mode in fp32."""
    if a.dtype == torch.float32:
        return a @ b
    return (a @ b).to(a.dtype)


def attention(q, keys, values, slot_tokens, seq_len, d_head, causal=True):
    """Scaled dot-product attention over per-slot queries (moe_layers.py:280-327).

    Slots must be chronological (slot s belongs to token s // k), as momha_forward produces.
    """
    require_dims(q.shape[1] == keys.shape[1] == values.shape[1], "projection widths", (q.shape[1],),
                 (keys.shape[1], values.shape[1]))
    if q.shape[1] % d_head:
        raise ValueError(f"projection width {q.shape[1]} is not divisible by d_head {d_head}")
    n = keys.shape[0]
    if n % seq_len:
        raise ValueError(f"token count {n} is not divisible by seq_len {seq_len}")
    k = q.shape[0] // n
    return _attn_core(q, keys, values, seq_len, d_head, k, causal)


def attention_backward(q, keys, values, slot_tokens, seq_len, d_head, causal, d_out):
    """(dq, dkeys, dvalues) by recomputation (moe_layers.py:330-377)."""
    n = keys.shape[0]
    k = q.shape[0] // n
    with torch.enable_grad():
        qv = q.detach().requires_grad_(True)
        kv = keys.detach().requires_grad_(True)
        vv = values.detach().requires_grad_(True)
        out = _attn_core(qv, kv, vv, seq_len, d_head, k, causal)
        dq, dk, dv = torch.autograd.grad(out, (qv, kv, vv), d_out.to(q.dtype))
    return dq, dk, dv


@dataclass
class MomhaContext:
    query_ctx: pl.LinearContext
    output_ctx: pl.LinearContext
    x: torch.Tensor
    q: torch.Tensor
    keys: torch.Tensor
    values: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    slot_tokens: torch.Tensor | None
    seq_len: int
    d_head: int
    causal: bool
    attn_graph: tuple | None = None   # (q, k, v leaves, output) of the bf16 training forward


@dataclass
class MomhaGradients:
    dx: torch.Tensor
    dwq: torch.Tensor
    dwk: torch.Tensor
    dwv: torch.Tensor
    dwo: torch.Tensor
    dp: torch.Tensor


def momha_forward(x, weights: MomhaWeights, routing: RoutingResult, order: GroupedOrder,
                  config: MomhaConfig, seq_len: int, *, training: bool = True,
                  tile: TileConfig | None = None, ledger=None):
    """Routed attention over flattened tokens (moe_layers.py:406-457).

    The two routed projections are ParallelLinear calls with chronological
    (scattered->scattered) layout, exactly the reference's :438-449.
    """
    n = x.shape[0]
    require_dims(x.shape[1] == config.d_model, "input width", tuple(x.shape), (config.d_model,))
    if n % seq_len:
        raise ValueError(f"token count {n} is not divisible by seq_len {seq_len}")
    if routing.num_tokens != n or routing.k != config.k:
        raise ValueError(f"routing covers {routing.num_tokens} tokens with k={routing.k}; "
                         f"expected {n} tokens with k={config.k}")
    keys = _mm(x, weights.wk)
    values = _mm(x, weights.wv)
    fused = (training and x.dtype == torch.bfloat16 and config.d_head % 8 == 0
             and (weights.wq.shape[2] % config.d_head) == 0)
    grouped = fused and _MOMHA_GROUPED
    # bf16 training: the slot rows around the attention core live in GROUPED
    # order — the query projection writes grouped rows (TMA slab stores), one
    # pass moves them into the core's head layout, one pass brings the core's
    # output back as grouped rows, and the output projection then reads them by
    # TMA (no row gather) and its backward stays in grouped order too
    heads_out = grouped and config.d_head % 64 == 0 and _MOMHA_HEADS_OUT
    if heads_out:
        # the query projection writes the attention core's head layout directly
        b_, kk_, dh_ = n // seq_len, config.k, config.d_head
        q = K.scatter2scatter_heads(x, weights.wq, order, kk_, False, batch=b_, seq_len=seq_len, k=kk_, d_head=dh_)
        query_ctx = pl.LinearContext(x=x, w=weights.wq, order=order, p=None, fan_out=kk_, x_was_grouped=False,
                                     y_was_grouped=True, y_hat=None)
    else:
        q_layout = SCATTERED_TO_GROUPED if grouped else SCATTERED_TO_SCATTERED
        q, query_ctx = pl.forward(x, weights.wq, order, p=None, fan_out=config.k, layout=q_layout,
                                  tile=tile, training=training, ledger=ledger, name="momha.query")
    attn_graph = None
    o_layout = SCATTERED_TO_SCATTERED
    if fused:
        # keep the attention core's autograd graph for the backward instead of
        # recomputing it (attention_backward, the reference's :330-377 form)
        kk, dh = config.k, config.d_head
        b, h = n // seq_len, weights.wq.shape[2] // dh
        if heads_out:
            qh = q
        elif grouped:
            qh = K.grouped_to_heads(q, order, kk, b, seq_len, dh)
        else:   # slot rows (b, S, k, h, d) -> heads (b, h*k, S, d) by 16-byte-element copies
            qh = _contig16(q.view(b, seq_len, kk, h, dh).permute(0, 3, 2, 1, 4)).view(b, h * kk, seq_len, dh)
        with torch.enable_grad():
            qv = qh.requires_grad_(True)
            kv = keys.view(b, seq_len, h, dh).transpose(1, 2).detach().requires_grad_(True)
            vv = values.view(b, seq_len, h, dh).transpose(1, 2).detach().requires_grad_(True)
            out = torch.nn.functional.scaled_dot_product_attention(qv, kv, vv, is_causal=config.causal,
                                                                   enable_gqa=kk > 1)
        attn_graph = (qv, kv, vv, out, (b, seq_len, kk, h, dh))
        if grouped:
            attn_out = K.heads_to_grouped(out.detach().contiguous(), order, kk)
            o_layout = GROUPED_TO_SCATTERED
        else:
            attn_out = _contig16(out.detach().view(b, h, kk, seq_len, dh).permute(0, 3, 2, 1, 4)).view(n * kk, h * dh)
    else:
        attn_out = attention(q, keys, values, None, seq_len, config.d_head, config.causal)
    y, output_ctx = pl.forward(attn_out, weights.wo, order, p=routing.p, fan_out=1,
                               layout=o_layout, tile=tile, training=training, ledger=ledger,
                               name="momha.output")
    if not training:
        return y, None
    return y, MomhaContext(query_ctx=query_ctx, output_ctx=output_ctx, x=x, q=q, keys=keys, values=values,
                           wk=weights.wk, wv=weights.wv, slot_tokens=None, seq_len=seq_len, attn_graph=attn_graph,
                           d_head=config.d_head, causal=config.causal)


def momha_backward(ctx: MomhaContext, dy, *, tile: TileConfig | None = None, ledger=None) -> MomhaGradients:
    """Gradients for routed attention; stops at dp (moe_layers.py:460-482)."""
    dx_heads = None
    if ctx.attn_graph is not None and ctx.output_ctx.x_was_grouped and _MOMHA_HEADS_OUT:
        _, _, _, _, (b, sl, kk, h, dh) = ctx.attn_graph
        if dh % 64 == 0:
            dx_heads = (b, sl, kk, dh)
    g_o = pl.backward(ctx.output_ctx, dy, tile=tile, ledger=ledger, name="momha.output", dx_heads=dx_heads)
    if ctx.attn_graph is not None:
        qv, kv, vv, out, (b, sl, kk, h, dh) = ctx.attn_graph
        ctx.attn_graph = None
        if dx_heads is not None:           # the input-gradient GEMM wrote the core's head layout
            d_out = g_o.dx
        elif ctx.output_ctx.x_was_grouped:   # the output projection's input gradient comes back as grouped rows
            d_out = K.grouped_to_heads(g_o.dx.to(out.dtype), ctx.output_ctx.order, kk, b, sl, dh)
        else:
            d_out = _contig16(g_o.dx.to(out.dtype).view(b, sl, kk, h, dh).permute(0, 3, 2, 1, 4)).view(b, h * kk, sl, dh)
        dqh, dkh, dvh = torch.autograd.grad(out, (qv, kv, vv), d_out)
        # the query gradient goes straight from the head layout to grouped rows:
        # the query projection's backward then reads it by TMA
        dq = K.heads_to_grouped(dqh.contiguous(), ctx.query_ctx.order, kk)
        ctx.query_ctx.y_was_grouped = True
        dk = _contig16(dkh.transpose(1, 2)).view(b * sl, h * dh)
        dv = _contig16(dvh.transpose(1, 2)).view(b * sl, h * dh)
    else:
        dq, dk, dv = attention_backward(ctx.q, ctx.keys, ctx.values, None, ctx.seq_len, ctx.d_head, ctx.causal,
                                        g_o.dx)
    g_q = pl.backward(ctx.query_ctx, dq, tile=tile, ledger=ledger, name="momha.query")
    x = ctx.x
    dwk = _mm(x.t(), dk)
    dwv = _mm(x.t(), dv)
    # dx = dx_q + dk Wk^T + dv Wv^T as one GEMM over the concatenated K/V gradients
    if x.dtype == torch.bfloat16:
        # dx = dx_q + [dk dv] [Wk Wv]^T in one GEMM with the sum in its epilogue
        dx = torch.addmm(g_q.dx, torch.cat([dk, dv], 1), torch.cat([ctx.wk, ctx.wv], 1).t())
    else:
        dx_kv = torch.cat([dk, dv], 1) @ torch.cat([ctx.wk, ctx.wv], 1).t()
        dx = (g_q.dx.float() + dx_kv.float()).to(x.dtype)
    return MomhaGradients(dx=dx, dwq=g_q.dw, dwk=dwk, dwv=dwv, dwo=g_o.dw, dp=g_o.dp)
