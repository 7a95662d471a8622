"""Padding-free grouped kernels over scattered or grouped row layouts (GPU).

Same API as the reference kernels.py (/root/reference/pkg/src/scattermlp/kernels.py):
scatter2scatter (:143-220), scatter_combine (:242-286), group (:289-326),
group_xty (:329-361), LayoutFlag + the four layout constants (:61-72),
TileConfig (:46-58), the MAC counter (:74-98) and the fault hook (:100-107).

Arguments are torch CUDA tensors: activations (rows, cols) in bfloat16 (the
tcgen05 product path), float32 (the check mode: 64-bit accumulation, one
rounding) or float64 (the reference's verification dtype), expert stacks
(E, d_in, d_out) of the same dtype, combine weights in float32 (float64 with
float64 storage).  Every call enqueues sm_100a kernels from libsmoe_b200.so on
the current stream; nothing here computes on the CPU and there is no fallback:
a bf16 call the tensor-core engine cannot take raises NotImplementedError.

TileConfig is accepted for API compatibility and ignored: the GPU kernels
choose their own tiles, and results never depend on tiling (the reference's
own invariant, kernels.py:46-49).
"""
from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field

import torch

from . import _lib
from . import launch_timer as _lt
from .errors import require_dims
from .router import GroupedOrder


def default_worker_count() -> int:
    env = os.environ.get("SCATTERMLP_WORKERS")
    if env is not None:
        n = int(env)
        if n < 1:
            raise ValueError(f"SCATTERMLP_WORKERS must be >= 1, got {n}")
        return n
    return os.cpu_count() or 1


@dataclass(frozen=True)
class TileConfig:
    """Reference blocking knobs (kernels.py:46-58); accepted, validated, unused on GPU."""

    tile_rows: int = 64
    tile_cols: int = 64
    tile_inner: int = 64
    worker_count: int = field(default_factory=default_worker_count)

    def __post_init__(self):
        for name in ("tile_rows", "tile_cols", "tile_inner", "worker_count"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")


@dataclass(frozen=True)
class LayoutFlag:
    """Whether the kernel's input/output rows are in grouped (bin) order."""

    grouped_in: bool = False
    grouped_out: bool = False


SCATTERED_TO_GROUPED = LayoutFlag(grouped_in=False, grouped_out=True)
GROUPED_TO_SCATTERED = LayoutFlag(grouped_in=True, grouped_out=False)
SCATTERED_TO_SCATTERED = LayoutFlag(grouped_in=False, grouped_out=False)
GROUPED_TO_GROUPED = LayoutFlag(grouped_in=True, grouped_out=True)

# ---- analytic MAC counter (kernels.py:74-98) and fault hook (:100-107) -------
_mac_lock = threading.Lock()
_mac_count = 0
_fault_inject = False
_engine = os.environ.get("SMOE_ENGINE", "auto")
# group() with fan-out > 1 walks source rows (smoe_group_inv) instead of grouped
# positions; SMOE_GROUP_BY_TOKEN=0 keeps the grouped-order walk (A/B)
_GROUP_BY_TOKEN = os.environ.get("SMOE_GROUP_BY_TOKEN", "1") != "0"
# scatter_combine: "auto" fuses the combine into the GEMM epilogue for k <= 2
# (bit-reproducible, no T*k buffer) and runs GEMM + combine for k > 2; "1"/"0" force
_COMBINE_FUSED = os.environ.get("SMOE_COMBINE_FUSED", "auto")


def reset_mac_count() -> None:
    global _mac_count
    with _mac_lock:
        _mac_count = 0


def mac_count() -> int:
    with _mac_lock:
        return _mac_count


def add_macs(n: int) -> None:
    global _mac_count
    with _mac_lock:
        _mac_count += int(n)


def _credit(order: GroupedOrder, d_in: int, d_out: int) -> None:
    # sum_e count_e * d_in * d_out == num_slots * d_in * d_out: padding-free.
    add_macs(order.num_slots * d_in * d_out)


def set_fault_injection(enabled: bool) -> None:
    """Test hook: corrupt one scatter2scatter output element per call."""
    global _fault_inject
    _fault_inject = bool(enabled)


def set_engine(name: str) -> None:
    """Select the GEMM engine: 'auto' (tcgen05 for bf16, SIMT for fp32), 'simt', 'tcgen05'."""
    global _engine
    if name not in _lib.ENGINE_IDS:
        raise ValueError(f"unknown engine {name!r}; choose from {sorted(_lib.ENGINE_IDS)}")
    _engine = name


def get_engine() -> str:
    return _engine


# ---- helpers -------------------------------------------------------------------

def _dtype_id(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SMOE_BF16
    if t.dtype == torch.float32:
        return _lib.SMOE_F32
    if t.dtype == torch.float64:
        return _lib.SMOE_F64
    raise ValueError(f"unsupported element type {t.dtype}; use bfloat16, float32 or float64")


def _wdtype(t: torch.Tensor) -> torch.dtype:
    """Element type of per-slot weights / dp for storage like t (include/smoe_b200.h smoe_dtype)."""
    return torch.float64 if t.dtype == torch.float64 else torch.float32


def _cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    return t if t.is_contiguous() else t.contiguous()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _engine_id(engine: str | None) -> int:
    return _lib.ENGINE_IDS[engine or _engine]


def _s2s_label(layout: LayoutFlag, transpose_w: bool, epi: int) -> str:
    lab = "scatter2scatter " + ("G" if layout.grouped_in else "S") + "->" + ("G" if layout.grouped_out else "S")
    if transpose_w:
        lab += " W^T"
    return lab + {_lib.EPI_NONE: "", _lib.EPI_ACT: " +act(pre,post)", _lib.EPI_ACT_GRAD: " *act'",
                  _lib.EPI_ACT_ONLY: " +act"}.get(epi, "")


# ---- kernels ---------------------------------------------------------------------

def scatter2scatter(
    x: torch.Tensor,
    w: torch.Tensor,
    order: GroupedOrder,
    fan_out: int,
    layout: LayoutFlag = SCATTERED_TO_SCATTERED,
    tile: TileConfig | None = None,
    *,
    transpose_w: bool = False,
    out: torch.Tensor | None = None,
    activation: str | None = None,
    act_out: torch.Tensor | None = None,
    act_grad_of: torch.Tensor | None = None,
    engine: str | None = None,
) -> torch.Tensor:
    """Fused gather -> per-expert linear transform -> scatter (kernels.py:143-220).

    Returns a T*k x d_out tensor in grouped order when layout.grouped_out else
    in scattered slot order.  Extensions beyond the reference (fused epilogues):
      activation + act_out: out holds the pre-activation, act_out = act(out)
        (the fusion of moe_layers.py:169-175);
      activation + act_grad_of: out = (x @ W) * act'(act_grad_of)  (moe_layers.py:205-206);
      activation alone: out = act(x @ W)  (inference, no pre-activation kept).
    """
    if fan_out < 1:
        raise ValueError(f"fan_out must be >= 1, got {fan_out}")
    num_slots = order.num_slots
    if w.dim() != 3:
        raise ValueError(f"expected a 3-D expert stack, got shape {tuple(w.shape)}")
    require_dims(order.num_experts == w.shape[0], "order bins vs expert stack",
                 (order.num_experts,), (w.shape[0],))
    d_in = w.shape[2] if transpose_w else w.shape[1]
    d_out = w.shape[1] if transpose_w else w.shape[2]
    require_dims(x.shape[1] == d_in, "input width vs expert weights", tuple(x.shape), (d_in, d_out))
    if layout.grouped_in:
        require_dims(x.shape[0] == num_slots, "grouped input rows vs slots", (x.shape[0],), (num_slots,))
    elif x.shape[0] * fan_out != num_slots:
        raise ValueError(
            f"scattered input rows ({x.shape[0]}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
    if w.dtype != x.dtype:
        raise ValueError(f"weight dtype {w.dtype} does not match input dtype {x.dtype}")
    if out is not None:
        require_dims(tuple(out.shape) == (num_slots, d_out), "out buffer", tuple(out.shape), (num_slots, d_out))
        if out.dtype != x.dtype:
            raise ValueError(f"out dtype {out.dtype} does not match input dtype {x.dtype}")
        if not out.is_contiguous():
            raise ValueError("out buffer must be contiguous")
    x = _cuda(x, "x")
    w = _cuda(w, "w")
    if out is None:
        out = torch.empty((num_slots, d_out), dtype=x.dtype, device=x.device)
    epi, act_id, aux = _lib.EPI_NONE, 0, None
    if activation is not None:
        if activation not in _lib.ACTIVATION_IDS:
            raise ValueError(f"unknown activation {activation!r}; choose from {sorted(_lib.ACTIVATION_IDS)}")
        act_id = _lib.ACTIVATION_IDS[activation]
        if act_out is not None and act_grad_of is not None:
            raise ValueError("activation takes at most one of act_out / act_grad_of")
        if act_out is None and act_grad_of is None:
            epi = _lib.EPI_ACT_ONLY
        elif act_out is not None:
            epi = _lib.EPI_ACT
            require_dims(tuple(act_out.shape) == (num_slots, d_out), "act_out buffer",
                         tuple(act_out.shape), (num_slots, d_out))
        else:
            epi = _lib.EPI_ACT_GRAD
            require_dims(tuple(act_grad_of.shape) == (num_slots, d_out), "act_grad_of",
                         tuple(act_grad_of.shape), (num_slots, d_out))
            aux = _cuda(act_grad_of, "act_grad_of")
    lib = _lib.load()
    t0 = _lt.begin()
    st = lib.smoe_scatter2scatter(
        x.data_ptr(), x.shape[0], w.data_ptr(), w.shape[0], w.shape[1], w.shape[2],
        order.o.data_ptr(), order.bin_offsets.data_ptr(), num_slots, fan_out,
        int(layout.grouped_in), int(layout.grouped_out), int(transpose_w), _dtype_id(x), epi, act_id,
        out.data_ptr(), _ptr(act_out), _ptr(aux), _engine_id(engine), _stream(x))
    _lt.end(_s2s_label(layout, transpose_w, epi), t0)
    _lib.check(st, "scatter2scatter")
    _credit(order, d_in, d_out)
    if _fault_inject and out.numel():
        out.view(-1)[0] += 0.01
    return out


def scatter_combine(
    x: torch.Tensor,
    w: torch.Tensor,
    order: GroupedOrder,
    fan_out: int,
    p_flat: torch.Tensor,
    combine_cols: int,
    grouped_in: bool,
    tile: TileConfig | None = None,
    *,
    engine: str | None = None,
) -> torch.Tensor:
    """scatter2scatter with the weighted slot-sum fused into the write (kernels.py:242-286).

    The T*k pre-combine buffer never exists: the per-slot products are scaled by
    p and accumulated into an fp32 (T, d_out) buffer, then rounded once.  bf16
    runs the tcgen05 GEMM with the scale-and-add in its epilogue (fp32 vector
    reductions; the k additions per token land in completion order, so results
    are bit-reproducible for k <= 2 and within fp32 rounding otherwise).
    """
    if fan_out < 1:
        raise ValueError(f"fan_out must be >= 1, got {fan_out}")
    num_slots = order.num_slots
    if num_slots % combine_cols:
        raise ValueError(f"combine width {combine_cols} must divide T*k ({num_slots})")
    require_dims(tuple(p_flat.shape) == (num_slots,), "combine weights", tuple(p_flat.shape), (num_slots,))
    d_in, d_out = w.shape[1], w.shape[2]
    require_dims(x.shape[1] == d_in, "input width vs expert weights", tuple(x.shape), (d_in, d_out))
    if grouped_in:
        require_dims(x.shape[0] == num_slots, "grouped input rows vs slots", (x.shape[0],), (num_slots,))
    elif x.shape[0] * fan_out != num_slots:
        raise ValueError(
            f"scattered input rows ({x.shape[0]}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
    x, w = _cuda(x, "x"), _cuda(w, "w")
    p32 = _cuda(p_flat.to(_wdtype(x)), "p_flat")
    rows = num_slots // combine_cols
    if (x.dtype == torch.bfloat16 and _COMBINE_FUSED != "1"
            and (engine or _engine) != "simt") or _COMBINE_FUSED == "0":
        # bf16: a scattered-output GEMM + the token-major combine.  The fused
        # combine epilogue (SMOE_COMBINE_FUSED=1) issues n*d_out fp32 L2
        # reductions, which cost more than the n-row round trip (C1 inference:
        # 11.15-11.36 vs 11.34-11.62 ms per forward; C2 layer 2: 3.06 + 0.48 vs
        # 4.13 ms), its fp32 accumulator is as large as the n-row buffer at
        # k = 2 (T*d*4 = T*k*d*2 B), and for k > 2 its additions land in
        # completion order (not bit-reproducible).
        y_hat = scatter2scatter(x, w, order, fan_out, LayoutFlag(grouped_in, False), engine=engine)
        return combine(p32.view(rows, combine_cols), y_hat)
    acc = torch.empty((rows, d_out), dtype=_wdtype(x), device=x.device)
    y = acc if x.dtype != torch.bfloat16 else torch.empty((rows, d_out), dtype=x.dtype, device=x.device)
    t0 = _lt.begin()
    st = _lib.load().smoe_scatter_combine(
        x.data_ptr(), x.shape[0], w.data_ptr(), w.shape[0], d_in, d_out, order.o.data_ptr(),
        order.bin_offsets.data_ptr(), num_slots, fan_out, p32.data_ptr(), combine_cols, int(grouped_in),
        _dtype_id(x), acc.data_ptr(), y.data_ptr(), _engine_id(engine), _stream(x))
    _lt.end("scatter_combine " + ("G" if grouped_in else "S") + "->combine", t0)
    _lib.check(st, "scatter_combine")
    _credit(order, d_in, d_out)
    return y


def group(
    x: torch.Tensor,
    order: GroupedOrder,
    weights: torch.Tensor | None = None,
    fan_out: int = 1,
    out: torch.Tensor | None = None,
) -> torch.Tensor:
    """Copy into grouped order: row i <- x[o[i] // fan_out] * weights[o[i]] (kernels.py:289-326)."""
    if fan_out < 1:
        raise ValueError(f"fan_out must be >= 1, got {fan_out}")
    num_slots = order.num_slots
    if x.shape[0] * fan_out != num_slots:
        raise ValueError(f"input rows ({x.shape[0]}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
    x = _cuda(x, "x")
    if weights is not None:
        require_dims(tuple(weights.shape) == (num_slots,), "slot weights", tuple(weights.shape), (num_slots,))
        weights = _cuda(weights.to(_wdtype(x)), "weights")
    if out is None:
        out = torch.empty((num_slots, x.shape[1]), dtype=x.dtype, device=x.device)
    else:
        require_dims(tuple(out.shape) == (num_slots, x.shape[1]), "out buffer", tuple(out.shape),
                     (num_slots, x.shape[1]))
        if out.dtype != x.dtype:
            raise ValueError(f"out dtype {out.dtype} does not match input dtype {x.dtype}")
    t0 = _lt.begin()
    if _GROUP_BY_TOKEN and 1 < fan_out <= 16 and order.inv is not None:
        # visited by source row: each x row read once, written to its k grouped positions
        st = _lib.load().smoe_group_inv(x.data_ptr(), x.shape[0], x.shape[1], order.inv.data_ptr(), fan_out,
                                        _ptr(weights), _dtype_id(x), out.data_ptr(), _stream(x))
    else:
        st = _lib.load().smoe_group(x.data_ptr(), x.shape[0], x.shape[1], order.o.data_ptr(), num_slots,
                                    fan_out, _ptr(weights), _dtype_id(x), out.data_ptr(), _stream(x))
    _lt.end("group", t0)
    _lib.check(st, "group")
    return out


def group_xty(
    xg: torch.Tensor,
    yg: torch.Tensor,
    order: GroupedOrder,
    tile: TileConfig | None = None,
    *,
    out: torch.Tensor | None = None,
    engine: str | None = None,
) -> torch.Tensor:
    """Per-expert Gram blocks dW[e] = Xg[bin e]^T @ Yg[bin e]; empty bin -> 0 (kernels.py:329-361)."""
    num_slots = order.num_slots
    require_dims(xg.shape[0] == num_slots, "grouped X rows vs slots", (xg.shape[0],), (num_slots,))
    require_dims(yg.shape[0] == num_slots, "grouped Y rows vs slots", (yg.shape[0],), (num_slots,))
    if xg.dtype != yg.dtype:
        raise ValueError(f"group_xty operands must share a dtype, got {xg.dtype} and {yg.dtype}")
    xg, yg = _cuda(xg, "xg"), _cuda(yg, "yg")
    d_in, d_out = xg.shape[1], yg.shape[1]
    e = order.num_experts
    if out is None:
        out = torch.empty((e, d_in, d_out), dtype=xg.dtype, device=xg.device)
    else:
        require_dims(tuple(out.shape) == (e, d_in, d_out), "dw buffer", tuple(out.shape), (e, d_in, d_out))
    t0 = _lt.begin()
    st = _lib.load().smoe_group_xty(xg.data_ptr(), yg.data_ptr(), order.bin_offsets.data_ptr(), e,
                                    num_slots, d_in, d_out, _dtype_id(xg), out.data_ptr(),
                                    _engine_id(engine), _stream(xg))
    _lt.end("group_xty", t0)
    _lib.check(st, "group_xty")
    _credit(order, d_in, d_out)
    return out


def scatter2scatter_scaled(
    x: torch.Tensor,
    w: torch.Tensor,
    order: GroupedOrder,
    fan_out: int,
    layout: LayoutFlag,
    *,
    row_scale: torch.Tensor,
    activation: str,
    out: torch.Tensor,
    act_out: torch.Tensor | None = None,
    act_grad_of: torch.Tensor | None = None,
    dp_partials: torch.Tensor | None = None,
    transpose_w: bool = False,
) -> torch.Tensor:
    """scatter2scatter with a routing-weight-scaled activation epilogue (bf16, tcgen05).

    act_out given: out = x @ W (pre-activation), act_out = s * act(out);
    activation="identity" (act = z, act' = 1) serves a plain routed linear with
    combine weights (parallel_linear.backward's dp-in-epilogue path);
    act_grad_of given: out = s * (x @ W) * act'(act_grad_of) and, when
    dp_partials ([n, dp_parts(d_out)] fp32) is given, the per-row partial dot
    products sum(acc * act(act_grad_of)) for the combine-weight gradient.
    s = row_scale[order.o[i]] for grouped row i (row_scale: one float per slot).
    """
    if (act_out is None) == (act_grad_of is None):
        raise ValueError("give exactly one of act_out / act_grad_of")
    if activation != "identity" and activation not in _lib.ACTIVATION_IDS:
        raise ValueError(f"unknown activation {activation!r}; choose from {sorted(_lib.ACTIVATION_IDS)}")
    act_id = _lib.ACT_IDENTITY if activation == "identity" else _lib.ACTIVATION_IDS[activation]
    if x.dtype != torch.bfloat16:
        raise ValueError("scaled epilogues run on the bf16 tensor-core engine")
    num_slots = order.num_slots
    d_in = w.shape[2] if transpose_w else w.shape[1]
    d_out = w.shape[1] if transpose_w else w.shape[2]
    require_dims(x.shape[1] == d_in, "input width vs expert weights", tuple(x.shape), (d_in, d_out))
    require_dims(tuple(out.shape) == (num_slots, d_out), "out buffer", tuple(out.shape), (num_slots, d_out))
    require_dims(tuple(row_scale.shape) == (num_slots,), "row scale", tuple(row_scale.shape), (num_slots,))
    x, w = _cuda(x, "x"), _cuda(w, "w")
    scale = _cuda(row_scale.to(torch.float32), "row_scale")
    epi = _lib.EPI_ACT_SCALED if act_out is not None else _lib.EPI_ACT_GRAD_SCALED
    parts = 0
    if dp_partials is not None:
        parts = _lib.load().smoe_dp_parts(d_out)
        require_dims(tuple(dp_partials.shape) == (num_slots, parts), "dp partials", tuple(dp_partials.shape),
                     (num_slots, parts))
    aux = None if act_grad_of is None else _cuda(act_grad_of, "act_grad_of")
    t0 = _lt.begin()
    st = _lib.load().smoe_scatter2scatter_scaled(
        x.data_ptr(), x.shape[0], w.data_ptr(), w.shape[0], w.shape[1], w.shape[2], order.o.data_ptr(),
        order.bin_offsets.data_ptr(), num_slots, fan_out, int(layout.grouped_in), int(layout.grouped_out),
        int(transpose_w), epi, act_id, scale.data_ptr(), out.data_ptr(), _ptr(act_out),
        _ptr(aux), _ptr(dp_partials), parts, _stream(x))
    _lt.end(_s2s_label(layout, transpose_w, _lib.EPI_ACT if act_out is not None else _lib.EPI_ACT_GRAD) + " scaled",
            t0)
    _lib.check(st, "scatter2scatter_scaled")
    _credit(order, d_in, d_out)
    return out


def heads_to_grouped(heads: torch.Tensor, order: GroupedOrder, k: int) -> torch.Tensor:
    """(n, h*d_head) slot rows in grouped order from the attention core's head layout.

    heads: (batch, h*k, seq_len, d_head) contiguous, head hh*k + j = choice j's head hh
    (moe_layers._attn_core); row i of the result is slot order.o[i]'s d_proj-wide row.
    """
    if heads.dim() != 4 or not heads.is_contiguous():
        raise ValueError("heads must be a contiguous (batch, heads, seq_len, d_head) tensor")
    b, hk, seq_len, dh = heads.shape
    if hk % k:
        raise ValueError(f"head count {hk} is not divisible by k={k}")
    n = order.num_slots
    require_dims(n == b * seq_len * k, "slots vs batch*seq_len*k", (n,), (b * seq_len * k,))
    heads = _cuda(heads, "heads")
    out = torch.empty((n, (hk // k) * dh), dtype=heads.dtype, device=heads.device)
    t0 = _lt.begin()
    st = _lib.load().smoe_heads_to_grouped(heads.data_ptr(), b, seq_len, k, hk // k, dh, order.o.data_ptr(), n,
                                           _dtype_id(heads), out.data_ptr(), _stream(heads))
    _lt.end("heads_to_grouped", t0)
    _lib.check(st, "heads_to_grouped")
    return out


def scatter2scatter_heads(
    x: torch.Tensor,
    w: torch.Tensor,
    order: GroupedOrder,
    fan_out: int,
    grouped_in: bool,
    *,
    batch: int,
    seq_len: int,
    k: int,
    d_head: int,
    transpose_w: bool = False,
    row_scale: torch.Tensor | None = None,
    act_grad_of: torch.Tensor | None = None,
    dp_partials: torch.Tensor | None = None,
) -> torch.Tensor:
    """scatter2scatter whose output goes straight into the attention core's head
    layout (batch, h*k, seq_len, d_head): output row i (slot order.o[i]) lands in
    heads hh*k + j of its token (bf16, tcgen05; d_head a multiple of 64).

    act_grad_of given (GROUPED rows, [n, d_out]): the routing-weight-scaled
    identity act-grad epilogue of parallel_linear's dp-in-epilogue backward —
    out = row_scale[o[i]] * (x @ W) and, with dp_partials, the partial dot
    products with act_grad_of's row i.
    """
    if x.dtype != torch.bfloat16:
        raise ValueError("head-layout output runs on the bf16 tensor-core engine")
    num_slots = order.num_slots
    d_in = w.shape[2] if transpose_w else w.shape[1]
    d_out = w.shape[1] if transpose_w else w.shape[2]
    require_dims(x.shape[1] == d_in, "input width vs expert weights", tuple(x.shape), (d_in, d_out))
    require_dims(num_slots == batch * seq_len * k, "slots vs batch*seq_len*k", (num_slots,), (batch * seq_len * k,))
    if d_out % d_head:
        raise ValueError(f"output width {d_out} is not divisible by d_head {d_head}")
    x, w = _cuda(x, "x"), _cuda(w, "w")
    heads = torch.empty((batch, (d_out // d_head) * k, seq_len, d_head), dtype=x.dtype, device=x.device)
    epi, scale_ptr, aux_ptr, parts, parts_ptr = _lib.EPI_NONE, None, None, 0, None
    if act_grad_of is not None:
        require_dims(tuple(act_grad_of.shape) == (num_slots, d_out), "act-grad operand", tuple(act_grad_of.shape),
                     (num_slots, d_out))
        scale = _cuda(row_scale.to(torch.float32), "row_scale").contiguous()
        aux = _cuda(act_grad_of, "act_grad_of").contiguous()
        epi, scale_ptr, aux_ptr = _lib.EPI_ACT_GRAD_SCALED, scale.data_ptr(), aux.data_ptr()
        if dp_partials is not None:
            parts = _lib.load().smoe_dp_parts(d_out)
            require_dims(tuple(dp_partials.shape) == (num_slots, parts), "dp partials", tuple(dp_partials.shape),
                         (num_slots, parts))
            parts_ptr = dp_partials.data_ptr()
    t0 = _lt.begin()
    st = _lib.load().smoe_scatter2scatter_heads(
        x.data_ptr(), x.shape[0], w.data_ptr(), w.shape[0], w.shape[1], w.shape[2], order.o.data_ptr(),
        order.bin_offsets.data_ptr(), num_slots, fan_out, int(grouped_in), int(transpose_w), epi,
        _lib.ACT_IDENTITY if act_grad_of is not None else 0, scale_ptr, aux_ptr, parts_ptr, parts, seq_len, k,
        d_head, heads.data_ptr(), _stream(x))
    _lt.end("scatter2scatter " + ("G" if grouped_in else "S") + "->heads" + (" W^T" if transpose_w else ""), t0)
    _lib.check(st, "scatter2scatter_heads")
    _credit(order, d_in, d_out)
    return heads


def grouped_to_heads(grouped: torch.Tensor, order: GroupedOrder, k: int, batch: int, seq_len: int,
                     d_head: int) -> torch.Tensor:
    """The attention core's head layout (batch, h*k, seq_len, d_head) from grouped
    slot rows (n, h*d_head) — the reverse of heads_to_grouped."""
    grouped = _cuda(grouped, "grouped").contiguous()
    n = order.num_slots
    require_dims(grouped.shape[0] == n == batch * seq_len * k, "grouped rows vs batch*seq_len*k",
                 (grouped.shape[0],), (batch * seq_len * k,))
    if grouped.shape[1] % d_head:
        raise ValueError(f"row width {grouped.shape[1]} is not divisible by d_head {d_head}")
    h = grouped.shape[1] // d_head
    heads = torch.empty((batch, h * k, seq_len, d_head), dtype=grouped.dtype, device=grouped.device)
    t0 = _lt.begin()
    st = _lib.load().smoe_grouped_to_heads(grouped.data_ptr(), batch, seq_len, k, h, d_head, order.o.data_ptr(), n,
                                           _dtype_id(grouped), heads.data_ptr(), _stream(grouped))
    _lt.end("grouped_to_heads", t0)
    _lib.check(st, "grouped_to_heads")
    return heads


def scale_grouped_rows(x_grouped: torch.Tensor, order: GroupedOrder, weights: torch.Tensor,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = x_grouped[i] * weights[o[i]] (group()'s weighting for rows already grouped)."""
    x = _cuda(x_grouped, "x_grouped").contiguous()
    require_dims(x.shape[0] == order.num_slots, "grouped rows vs slots", (x.shape[0],), (order.num_slots,))
    w = _cuda(weights.reshape(-1).to(_wdtype(x)), "weights").contiguous()
    if out is None:
        out = torch.empty_like(x)
    t0 = _lt.begin()
    st = _lib.load().smoe_scale_grouped_rows(x.data_ptr(), x.shape[1], order.o.data_ptr(), x.shape[0], w.data_ptr(),
                                             _dtype_id(x), out.data_ptr(), _stream(x))
    _lt.end("scale_grouped_rows", t0)
    _lib.check(st, "scale_grouped_rows")
    return out


def dp_parts(d_out: int) -> int:
    return int(_lib.load().smoe_dp_parts(d_out))


def dp_from_partials(partials: torch.Tensor, order: GroupedOrder, s: int, j: int) -> torch.Tensor:
    """dp (s, j) float32 from the [n, parts] partial dot products of grouped rows."""
    dp = torch.empty((s, j), dtype=torch.float32, device=partials.device)
    t0 = _lt.begin()
    st = _lib.load().smoe_dp_from_partials(partials.data_ptr(), partials.shape[0], partials.shape[1],
                                           order.o.data_ptr(), dp.data_ptr(), _stream(partials))
    _lt.end("dp_from_partials", t0)
    _lib.check(st, "dp_from_partials")
    return dp


def group_xty_scattered(
    x: torch.Tensor,
    y: torch.Tensor,
    order: GroupedOrder,
    *,
    x_fan_out: int = 1,
    y_fan_out: int = 1,
    x_grouped: bool = False,
    y_grouped: bool = False,
    out: torch.Tensor | None = None,
    engine: str | None = None,
) -> torch.Tensor:
    """group_xty(group(x, fan_out=x_fan_out), group(y, fan_out=y_fan_out)) without the grouped copies.

    Row i of a bin reads x[order.o[i] // x_fan_out] (x[i] when x_grouped), likewise y:
    the reference's parallel_linear.py:224-234 (group + group_xty) fused into the
    GEMM's operand loads.
    """
    num_slots = order.num_slots
    for name, a, f, grouped in (("x", x, x_fan_out, x_grouped), ("y", y, y_fan_out, y_grouped)):
        if f < 1:
            raise ValueError(f"{name}_fan_out must be >= 1, got {f}")
        want = num_slots if grouped else num_slots // f
        if a.shape[0] != want or (not grouped and a.shape[0] * f != num_slots):
            raise ValueError(f"{name} rows ({a.shape[0]}) do not cover the {num_slots} slots "
                             f"({'grouped' if grouped else f'fan_out {f}'})")
    if x.dtype != y.dtype:
        raise ValueError(f"group_xty operands must share a dtype, got {x.dtype} and {y.dtype}")
    x, y = _cuda(x, "x"), _cuda(y, "y")
    d_in, d_out = x.shape[1], y.shape[1]
    e = order.num_experts
    if out is None:
        out = torch.empty((e, d_in, d_out), dtype=x.dtype, device=x.device)
    else:
        require_dims(tuple(out.shape) == (e, d_in, d_out), "dw buffer", tuple(out.shape), (e, d_in, d_out))
    t0 = _lt.begin()
    st = _lib.load().smoe_group_xty_scattered(
        x.data_ptr(), x.shape[0], x_fan_out, int(x_grouped), y.data_ptr(), y.shape[0], y_fan_out, int(y_grouped),
        order.o.data_ptr(), order.bin_offsets.data_ptr(), e, num_slots, d_in, d_out, _dtype_id(x),
        out.data_ptr(), _engine_id(engine), _stream(x))
    _lt.end("group_xty " + ("G" if x_grouped else "S") + ("G" if y_grouped else "S"), t0)
    _lib.check(st, "group_xty_scattered")
    _credit(order, d_in, d_out)
    return out


# ---- row kernels used by parallel_linear (not in the reference's kernels.py) ----

def combine(p: torch.Tensor, y_hat: torch.Tensor, out: torch.Tensor | None = None,
            inverse: torch.Tensor | None = None) -> torch.Tensor:
    """Y[s] = sum_i p[s, i] * Y_hat[s*j + i]  (parallel_linear.py:69-73).

    inverse: Y_hat holds the slot rows in grouped order (a grouped-output
    GEMM's layout) and slot r is row inverse[r]; same result bit for bit."""
    s, j = p.shape
    y_hat = _cuda(y_hat, "y_hat")
    p32 = _cuda(p.to(_wdtype(y_hat)), "p")
    if out is None:
        out = torch.empty((s, y_hat.shape[1]), dtype=y_hat.dtype, device=y_hat.device)
    t0 = _lt.begin()
    if inverse is not None:
        inv = _cuda(inverse, "inverse").to(torch.int32).contiguous()
        require_dims(inv.numel() == s * j == y_hat.shape[0], "inverse vs slot rows", (inv.numel(),), (s * j,))
        st = _lib.load().smoe_combine_grouped(y_hat.data_ptr(), inv.data_ptr(), p32.data_ptr(), s, j,
                                              y_hat.shape[1], _dtype_id(y_hat), out.data_ptr(), _stream(y_hat))
    else:
        st = _lib.load().smoe_combine(y_hat.data_ptr(), p32.data_ptr(), s, j, y_hat.shape[1],
                                      _dtype_id(y_hat), out.data_ptr(), _stream(y_hat))
    _lt.end("combine", t0)
    _lib.check(st, "combine")
    return out


def combine_grad_p(dy: torch.Tensor, y_hat: torch.Tensor, s: int, j: int,
                   inverse: torch.Tensor | None = None) -> torch.Tensor:
    """dp[s, i] = <dY[s], Y_hat[s*j + i]>  (parallel_linear.py:198-206), float32.

    inverse: Y_hat holds the slot rows in grouped order (slot r is row inverse[r])."""
    dy, y_hat = _cuda(dy, "dy"), _cuda(y_hat, "y_hat")
    dp = torch.empty((s, j), dtype=_wdtype(dy), device=dy.device)
    t0 = _lt.begin()
    if inverse is not None:
        inv = _cuda(inverse, "inverse").to(torch.int32).contiguous()
        require_dims(inv.numel() == s * j == y_hat.shape[0], "inverse vs slot rows", (inv.numel(),), (s * j,))
        st = _lib.load().smoe_combine_grad_p_grouped(dy.data_ptr(), y_hat.data_ptr(), inv.data_ptr(), s, j,
                                                     dy.shape[1], _dtype_id(dy), dp.data_ptr(), _stream(dy))
    else:
        st = _lib.load().smoe_combine_grad_p(dy.data_ptr(), y_hat.data_ptr(), s, j, dy.shape[1],
                                             _dtype_id(dy), dp.data_ptr(), _stream(dy))
    _lt.end("combine_grad_p", t0)
    _lib.check(st, "combine_grad_p")
    return dp


def fanout_reduce(slot_grads: torch.Tensor, fan_out: int, out: torch.Tensor | None = None,
                  inverse: torch.Tensor | None = None) -> torch.Tensor:
    """dX[t] = sum_j G[t*fan_out + j]  (parallel_linear.py:259-266).

    inverse: G holds the slot rows in grouped order (slot r is row inverse[r])."""
    g = _cuda(slot_grads, "slot_grads")
    t = g.shape[0] // fan_out
    if out is None:
        out = torch.empty((t, g.shape[1]), dtype=g.dtype, device=g.device)
    t0 = _lt.begin()
    if inverse is not None:
        inv = _cuda(inverse, "inverse").to(torch.int32).contiguous()
        require_dims(inv.numel() == g.shape[0], "inverse vs slot rows", (inv.numel(),), (g.shape[0],))
        st = _lib.load().smoe_fanout_reduce_grouped(g.data_ptr(), inv.data_ptr(), t, fan_out, g.shape[1],
                                                    _dtype_id(g), out.data_ptr(), _stream(g))
    else:
        st = _lib.load().smoe_fanout_reduce(g.data_ptr(), t, fan_out, g.shape[1], _dtype_id(g),
                                            out.data_ptr(), _stream(g))
    _lt.end("fanout_reduce", t0)
    _lib.check(st, "fanout_reduce")
    return out


def activation_kernel(x: torch.Tensor, name: str, derivative: bool,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """act(x) or act'(x), fp32 math, rounded once (moe_layers.py:75-83)."""
    if name not in _lib.ACTIVATION_IDS:
        raise ValueError(f"unknown activation {name!r}; choose from {sorted(_lib.ACTIVATION_IDS)}")
    x = _cuda(x, "x")
    if out is None:
        out = torch.empty_like(x)
    t0 = _lt.begin()
    st = _lib.load().smoe_apply_activation(x.data_ptr(), x.numel(), _lib.ACTIVATION_IDS[name],
                                           int(derivative), _dtype_id(x), out.data_ptr(), _stream(x))
    _lt.end("activation", t0)
    _lib.check(st, "activation")
    return out
