"""Top-k routing and the grouped execution order, on the GPU.

Mirrors router.py of the reference (/root/reference/pkg/src/scattermlp/router.py):
RoutingResult (:22-77), GroupedOrder (:80-116), gate_forward / softmax_rows /
topk_select (:119-151), compute_grouped_order (:154-164), gate_backward
(:167-188), assignment_routing (:191-218).

The hot-path piece is compute_grouped_order, which runs the stable counting
sort of csrc/sort.cu (K1) and is bit-exact against numpy's stable argsort.
It also produces the north_star names of upstream ScatterMoE:
``flatten_and_sort(expert_idxs) -> (sorted_expert_idxs, sorted_scattered_idxs)``
and the expert offsets (= GroupedOrder.bin_offsets[1:]).

Index tensors produced on the device are int32 (T*k < 2^31); compare against
the reference after casting to int64.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib
from . import launch_timer as _lt
from .errors import require_dims


def _stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass(frozen=True, eq=False)
class RoutingResult:
    """Selected experts and their combine weights for each token (router.py:22-36).

    expert_idx: (T, k) int64, distinct ids per row.
    p: (T, k) float32 combine weights aligned with expert_idx.
    gate_full: (T, E) full gate probabilities.
    renormalized: whether p rows were rescaled to sum to one.
    """

    expert_idx: torch.Tensor
    p: torch.Tensor
    gate_full: torch.Tensor
    renormalized: bool = True
    validate: bool = field(default=True, repr=False)

    def __post_init__(self):
        require_dims(tuple(self.expert_idx.shape) == tuple(self.p.shape), "expert_idx vs p",
                     self.expert_idx.shape, self.p.shape)
        require_dims(self.gate_full.shape[0] == self.expert_idx.shape[0], "gate rows vs routed rows",
                     self.gate_full.shape, self.expert_idx.shape)
        t, k = self.expert_idx.shape
        e = self.gate_full.shape[1]
        if k < 1 or k > e:
            raise ValueError(f"k must be in [1, E]; got k={k}, E={e}")
        if not self.validate or t == 0:
            return
        # Same checks as router.py:49-60, vectorised (one host sync).
        lo, hi = int(self.expert_idx.min()), int(self.expert_idx.max())
        if lo < 0 or hi >= e:
            raise ValueError(f"expert ids must lie in [0, {e}); got range [{lo}, {hi}]")
        srt = torch.sort(self.expert_idx, dim=1).values
        dup = (srt[:, 1:] == srt[:, :-1]).any(dim=1)
        if bool(dup.any()):
            row = int(torch.nonzero(dup)[0, 0])
            raise ValueError(f"duplicate expert id in row {row}: {self.expert_idx[row].tolist()}")
        if self.renormalized:
            sums = self.p.to(torch.float64).sum(dim=1)
            if not bool(torch.allclose(sums, torch.ones_like(sums), atol=1e-6, rtol=0)):
                raise ValueError("renormalized combine weights must sum to 1 per row")

    @property
    def num_tokens(self) -> int:
        return self.expert_idx.shape[0]

    @property
    def k(self) -> int:
        return self.expert_idx.shape[1]

    @property
    def num_experts(self) -> int:
        return self.gate_full.shape[1]

    @property
    def p_flat(self) -> torch.Tensor:
        """Combine weights indexed by scattered slot (token-major), router.py:74-77."""
        return self.p.reshape(-1)


@dataclass(frozen=True, eq=False)
class GroupedOrder:
    """Stable grouping of the T*k scattered slots by expert id (router.py:80-116).

    o[i] is the scattered slot held at grouped position i ("sorted_scattered_idxs");
    positions [bin_offsets[e], bin_offsets[e+1]) form expert e's bin.
    sorted_expert_idxs and inv (scattered slot -> grouped position) come from the
    same sort kernel and are kept for the EP dispatch and the tests.
    """

    o: torch.Tensor
    bin_offsets: torch.Tensor
    sorted_expert_idxs: torch.Tensor | None = None
    inv: torch.Tensor | None = field(default=None, repr=False)
    validate: bool = field(default=True, repr=False)

    def __post_init__(self):
        if self.bin_offsets.dim() != 1 or self.bin_offsets.numel() < 2:
            raise ValueError("bin_offsets must hold E+1 entries")
        if self.validate:
            off = self.bin_offsets.to("cpu", torch.int64)
            if int(off[0]) != 0 or int(off[-1]) != self.o.numel():
                raise ValueError("bin_offsets must start at 0 and end at T*k")
            if bool((off[1:] < off[:-1]).any()):
                raise ValueError("bin_offsets must be non-decreasing")

    @property
    def num_slots(self) -> int:
        return self.o.numel()

    @property
    def num_experts(self) -> int:
        return self.bin_offsets.numel() - 1

    @property
    def bin_counts(self) -> torch.Tensor:
        return self.bin_offsets[1:] - self.bin_offsets[:-1]

    @property
    def expert_offsets(self) -> torch.Tensor:
        """Upstream ScatterMoE's expert_offsets: the E bin END offsets."""
        return self.bin_offsets[1:]

    def inverse(self) -> torch.Tensor:
        """Map scattered slot -> grouped position (router.py:112-116)."""
        if self.inv is not None:
            return self.inv
        inv = torch.empty_like(self.o)
        inv[self.o.long()] = torch.arange(self.o.numel(), dtype=self.o.dtype, device=self.o.device)
        return inv


def _sort_ids(flat_ids: torch.Tensor, num_experts: int):
    """Run K1 on a flat int64 CUDA tensor; returns (o, sorted_ids, offsets, inverse)."""
    if not flat_ids.is_cuda:
        raise ValueError("expert ids must live on a CUDA device (no CPU path exists)")
    lib = _lib.load()
    ids = flat_ids.contiguous()
    if ids.dtype != torch.int64:
        ids = ids.to(torch.int64)
    n = ids.numel()
    dev = ids.device
    o = torch.empty(n, dtype=torch.int32, device=dev)
    sorted_ids = torch.empty(n, dtype=torch.int32, device=dev)
    inv = torch.empty(n, dtype=torch.int32, device=dev)
    offsets = torch.empty(num_experts + 1, dtype=torch.int32, device=dev)
    ws_bytes = lib.smoe_route_sort_workspace_bytes(n, num_experts)
    ws = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        t0 = _lt.begin()
        st = lib.smoe_route_sort(ids.data_ptr(), n, num_experts, o.data_ptr(), sorted_ids.data_ptr(),
                                 offsets.data_ptr(), inv.data_ptr(), ws.data_ptr(), ws_bytes,
                                 _stream_ptr(dev))
        _lt.end("route_sort", t0)
    _lib.check(st, "compute_grouped_order")
    return o, sorted_ids, offsets, inv


def compute_grouped_order(routing: RoutingResult, num_experts: int | None = None) -> GroupedOrder:
    """Group the T*k scattered slots by expert id, stable by slot index (router.py:154-164)."""
    e = routing.num_experts if num_experts is None else num_experts
    if e < routing.num_experts:
        raise ValueError(f"num_experts={e} smaller than routed id space {routing.num_experts}")
    o, sorted_ids, offsets, inv = _sort_ids(routing.expert_idx.reshape(-1), e)
    return GroupedOrder(o=o, bin_offsets=offsets, sorted_expert_idxs=sorted_ids, inv=inv, validate=False)


def flatten_and_sort(expert_idxs: torch.Tensor, num_experts: int | None = None,
                     return_offsets: bool = False):
    """Upstream ScatterMoE entry point: flatten (T, k) ids and stably sort them.

    Returns (sorted_expert_idxs, sorted_scattered_idxs) and, with
    return_offsets, also expert_offsets (the E bin end offsets).
    """
    if num_experts is None:
        num_experts = int(expert_idxs.max()) + 1 if expert_idxs.numel() else 1
    o, sorted_ids, offsets, _ = _sort_ids(expert_idxs.reshape(-1), num_experts)
    if return_offsets:
        return sorted_ids, o, offsets[1:]
    return sorted_ids, o


# ---- gate (outside the ParallelLinear hot path; torch glue) -----------------

def _softmax_rows64(z: torch.Tensor) -> torch.Tensor:
    z = z - z.max(dim=1, keepdim=True).values
    ez = torch.exp(z)
    return ez / ez.sum(dim=1, keepdim=True)


def gate_forward(x: torch.Tensor, w_g: torch.Tensor) -> torch.Tensor:
    """Row softmax of x @ w_g in float64, rounded to x's dtype (router.py:119-123)."""
    require_dims(x.shape[1] == w_g.shape[0], "gate matmul", x.shape, w_g.shape)
    logits = x.to(torch.float64) @ w_g.to(torch.float64)
    return _softmax_rows64(logits).to(torch.float32)


def gate_topk(x: torch.Tensor, w_g: torch.Tensor, k: int, renormalize: bool = True) -> RoutingResult:
    """topk_select(gate_forward(x, w_g), k) as one kernel (router.py:119-151).

    csrc/router.cu router_gate_kernel: the gate GEMM accumulated in float64 (the
    logits are never rounded), softmax in float64 rounded once to float32, the
    stable top-k on the float32 gates and the float64 renormalisation; the ids
    it writes go straight to compute_grouped_order.  x: (T, d_model) bf16 or
    float32 CUDA tensor; w_g: (d_model, E), used in float32.
    """
    require_dims(x.dim() == 2 and w_g.dim() == 2 and x.shape[1] == w_g.shape[0], "gate matmul", tuple(x.shape),
                 tuple(w_g.shape))
    t, e = x.shape[0], w_g.shape[1]
    if not 1 <= k <= e:
        raise ValueError(f"k must be in [1, E]; got k={k}, E={e}")
    if not x.is_cuda:
        raise ValueError("x must be a CUDA tensor (there is no CPU path)")
    if x.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError(f"x must be bfloat16 or float32, got {x.dtype}")
    x = x.contiguous()
    wg = w_g.to(device=x.device, dtype=torch.float32).contiguous()
    gate = torch.empty((t, e), dtype=torch.float32, device=x.device)
    idx = torch.empty((t, k), dtype=torch.int64, device=x.device)
    p = torch.empty((t, k), dtype=torch.float32, device=x.device)
    t0 = _lt.begin()
    st = _lib.load().smoe_router_gate(x.data_ptr(), _lib.SMOE_BF16 if x.dtype == torch.bfloat16 else _lib.SMOE_F32,
                                      wg.data_ptr(), t, x.shape[1], e, k, int(renormalize), gate.data_ptr(),
                                      idx.data_ptr(), p.data_ptr(), _stream_ptr(x.device))
    _lt.end("router_gate", t0)
    _lib.check(st, "gate_topk")
    return RoutingResult(expert_idx=idx, p=p, gate_full=gate, renormalized=renormalize, validate=False)


def softmax_rows(logits: torch.Tensor) -> torch.Tensor:
    """Stable row softmax (router.py:126-128)."""
    return _softmax_rows64(logits.to(torch.float64)).to(logits.dtype)


def _router_kernel(inp: torch.Tensor, k: int, renormalize: bool, apply_softmax: bool):
    """csrc/router.cu: (gate, expert_idx, p) for a CUDA [T, E] float32 input."""
    t, e = inp.shape
    inp = inp.to(torch.float32).contiguous()
    idx = torch.empty((t, k), dtype=torch.int64, device=inp.device)
    p = torch.empty((t, k), dtype=torch.float32, device=inp.device)
    gate = torch.empty_like(inp) if apply_softmax else inp
    t0 = _lt.begin()
    st = _lib.load().smoe_router_topk(inp.data_ptr(), t, e, k, int(apply_softmax), int(renormalize),
                                      gate.data_ptr() if apply_softmax else None, idx.data_ptr(), p.data_ptr(),
                                      _stream_ptr(inp.device))
    _lt.end("router_topk", t0)
    _lib.check(st, "router_topk")
    return gate, idx, p


def route(logits: torch.Tensor, k: int, renormalize: bool = True) -> RoutingResult:
    """Fused softmax + stable top-k + renormalisation of float32 logits (one kernel).

    Equivalent to topk_select(softmax_rows(logits), k) (router.py:126-151) with
    the softmax evaluated in float64 and rounded once, as the reference does.
    """
    t, e = logits.shape
    if not 1 <= k <= e:
        raise ValueError(f"k must be in [1, E]; got k={k}, E={e}")
    if not logits.is_cuda:
        return topk_select(softmax_rows(logits.to(torch.float32)), k, renormalize)
    gate, idx, p = _router_kernel(logits, k, renormalize, apply_softmax=True)
    return RoutingResult(expert_idx=idx, p=p, gate_full=gate, renormalized=renormalize, validate=False)


def topk_select(gate: torch.Tensor, k: int, renormalize: bool = True) -> RoutingResult:
    """Each row's k largest gates; ties toward the lower expert id (router.py:137-151).

    CUDA inputs run the router kernel (csrc/router.cu, k <= 8); CPU tensors use
    torch ops (host-side utilities and tests).
    """
    t, e = gate.shape
    if not 1 <= k <= e:
        raise ValueError(f"k must be in [1, E]; got k={k}, E={e}")
    if gate.is_cuda and k <= 8:
        _, idx, p = _router_kernel(gate, k, renormalize, apply_softmax=False)
        return RoutingResult(expert_idx=idx, p=p, gate_full=gate, renormalized=renormalize, validate=False)
    order = torch.sort(-gate, dim=1, stable=True).indices
    idx = order[:, :k].to(torch.int64).contiguous()
    sel = torch.gather(gate, 1, idx)
    if renormalize:
        s64 = sel.to(torch.float64)
        p = (s64 / s64.sum(dim=1, keepdim=True)).to(torch.float32)
    else:
        p = sel.to(torch.float32).clone()
    return RoutingResult(expert_idx=idx, p=p.contiguous(), gate_full=gate, renormalized=renormalize)


def gate_backward(routing: RoutingResult, grad_p: torch.Tensor) -> torch.Tensor:
    """Gradient wrt gate logits given dL/dp (router.py:167-188); router kernel on CUDA."""
    require_dims(tuple(grad_p.shape) == tuple(routing.p.shape), "grad_p vs p", grad_p.shape, routing.p.shape)
    if routing.gate_full.is_cuda:
        t, e = routing.gate_full.shape
        gate = routing.gate_full.to(torch.float32).contiguous()
        gp = grad_p.to(torch.float32).contiguous()
        idx = routing.expert_idx.to(torch.int64).contiguous()
        dz = torch.empty_like(gate)
        st = _lib.load().smoe_router_backward(gate.data_ptr(), idx.data_ptr(), gp.data_ptr(), t, e, routing.k,
                                              int(routing.renormalized), dz.data_ptr(), _stream_ptr(gate.device))
        _lib.check(st, "router_backward")
        return dz.to(routing.gate_full.dtype)
    g = routing.gate_full.to(torch.float64)
    dp = grad_p.to(torch.float64)
    sel = routing.expert_idx
    gsel = torch.gather(g, 1, sel)
    if routing.renormalized:
        s = gsel.sum(dim=1, keepdim=True)
        p = gsel / s
        dgsel = (dp - (dp * p).sum(dim=1, keepdim=True)) / s
    else:
        dgsel = dp
    dg = torch.zeros_like(g).scatter_(1, sel, dgsel)
    dz = g * (dg - (dg * g).sum(dim=1, keepdim=True))
    return dz.to(routing.gate_full.dtype)


def assignment_routing(expert_idx, num_experts: int, p=None, dtype=torch.float32,
                       device=None) -> RoutingResult:
    """RoutingResult from explicit assignments (router.py:191-218)."""
    idx = torch.as_tensor(expert_idx, dtype=torch.int64, device=device)
    if idx.dim() != 2:
        raise ValueError(f"expert_idx must be (T, k), got shape {tuple(idx.shape)}")
    if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= num_experts):
        raise ValueError(f"expert ids must lie in [0, {num_experts}); got range "
                         f"[{int(idx.min())}, {int(idx.max())}]")
    t, k = idx.shape
    if p is None:
        p = torch.full((t, k), 1.0 / k, dtype=dtype, device=idx.device)
    else:
        p = torch.as_tensor(p, dtype=dtype, device=idx.device)
        sums = p.to(torch.float64).sum(dim=1, keepdim=True)
        if not bool(torch.allclose(sums, torch.ones_like(sums), atol=1e-6, rtol=0)):
            p = (p.to(torch.float64) / sums).to(dtype)
    gate = torch.zeros((t, num_experts), dtype=dtype, device=idx.device)
    gate.scatter_(1, idx, p)
    return RoutingResult(expert_idx=idx.contiguous(), p=p.contiguous(), gate_full=gate, renormalized=True)
