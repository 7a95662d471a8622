"""Expert parallelism (EP) for the SMoE MLP: experts sharded over the GPUs of one box.

SURVEY.md §8(e).  The reference has no multi-device code; this is
the B200 build's one multi-GPU strategy.  Rank r owns the contiguous expert
range [r*E_l, (r+1)*E_l) (E_l = E / G) and its W1/W2 slices.  Per forward:

  1. K1 sort of the local routing over the GLOBAL expert ids.  Because expert
     ownership is contiguous, the grouped order is already rank-major: the rows
     for rank q are grouped positions [off[q*E_l], off[(q+1)*E_l]) — no second
     sort.
  2. pack:  send = group(X, o, fan_out=k)            (kernels.py:289-326)
  3. all-to-all of the per-expert counts (G x E_l), then all-to-all-v of the
     packed rows over NCCL (NVLink / NVSwitch).
  4. the receiver's local grouped order is a counts-only interleave (expert-major,
     then source rank, then source order) — identical row order to a single-GPU
     run on the concatenated batch, so outputs and dW are bit-identical to it.
  5. local expert MLP on the received rows (S->G layer 1 with fused activation,
     G->S layer 2 back to receive order, no combine).
  6. reverse all-to-all-v; the source un-permutes with the inverse order and
     applies the routing-weighted combine, keeping Y_hat for dp.
Backward mirrors it: dp and the p-weighted group of dY at the source, dispatch,
local backward (dW stays local: no all-reduce for expert weights), return the
slot input-gradients, un-permute and fan-out reduce at the source.

The local compute and the pack/unpack row ops go through an ``ops`` object.
The default is :class:`CudaOps` (the sm_100a kernels of libsmoe_b200.so); the
CPU multi-process tests inject a torch reference to exercise the
communication and index algebra with the gloo backend.  There is no CPU
fallback in the product path.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import kernels as K
from .kernels import GROUPED_TO_GROUPED, GROUPED_TO_SCATTERED, SCATTERED_TO_GROUPED
from .router import GroupedOrder, RoutingResult, compute_grouped_order


# ---------------------------------------------------------------------------
# index algebra (device-agnostic torch; int64 on host-side, int32 for kernels)

def local_order_from_counts(counts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Grouped order of the received rows from the (G sources x E_l experts) counts.

    Received rows are laid out source-major (each source's segment in its own
    expert-major grouped order).  The local grouped order is expert-major, then
    source, then the source's order.  Returns (o_loc int64 [n_recv], offsets int64 [E_l+1]).
    """
    g, e_l = counts.shape
    c = counts.to(torch.int64)
    flat = c.reshape(-1)
    recv_base = (torch.cumsum(flat, 0) - flat).reshape(g, e_l)       # start of (s, e) in recv layout
    lengths = c.t().reshape(-1)                                        # expert-major (e, s)
    starts = recv_base.t().reshape(-1)
    total = int(lengths.sum())
    seg_start_pos = torch.cumsum(lengths, 0) - lengths
    within = torch.arange(total, device=counts.device) - torch.repeat_interleave(seg_start_pos, lengths)
    o_loc = torch.repeat_interleave(starts, lengths) + within
    offsets = torch.zeros(e_l + 1, dtype=torch.int64, device=counts.device)
    offsets[1:] = torch.cumsum(c.sum(0), 0)
    return o_loc, offsets


def send_counts(order: GroupedOrder, world: int) -> torch.Tensor:
    """(G x E_l) per-destination, per-local-expert row counts from the global bins."""
    e = order.num_experts
    if e % world:
        raise ValueError(f"num_experts={e} must be divisible by the EP world size {world}")
    return order.bin_counts.to(torch.int64).reshape(world, e // world)


# ---------------------------------------------------------------------------
# compute backends

class CudaOps:
    """Routing sort, pack/unpack rows and the local expert MLP on the sm_100a kernels."""

    @staticmethod
    def order(routing: RoutingResult, num_experts: int) -> GroupedOrder:
        return compute_grouped_order(routing, num_experts)

    @staticmethod
    def group(x, order_o32, fan_out, weights=None):
        o = GroupedOrder(o=order_o32, bin_offsets=torch.zeros(2, dtype=torch.int32, device=x.device), validate=False)
        return K.group(x, o, weights=weights, fan_out=fan_out)

    @staticmethod
    def combine(p, y_hat):
        return K.combine(p, y_hat)

    @staticmethod
    def combine_grad_p(dy, y_hat, s, j):
        return K.combine_grad_p(dy, y_hat, s, j)

    @staticmethod
    def fanout_reduce(g, fan_out):
        return K.fanout_reduce(g, fan_out)

    @staticmethod
    def local_forward(r, w1, w2, o_loc, off_loc, activation):
        order = GroupedOrder(o=o_loc.to(torch.int32), bin_offsets=off_loc.to(torch.int32), validate=False)
        n, de = o_loc.numel(), w1.shape[2]
        h_pre = torch.empty((n, de), dtype=r.dtype, device=r.device)
        h = torch.empty_like(h_pre)
        K.scatter2scatter(r, w1, order, 1, SCATTERED_TO_GROUPED, out=h_pre, activation=activation, act_out=h)
        y = K.scatter2scatter(h, w2, order, 1, GROUPED_TO_SCATTERED)
        return y, (order, h_pre, h)

    @staticmethod
    def local_backward(r, w1, w2, saved, dy, activation):
        order, h_pre, h = saved
        gdy = K.group(dy, order, fan_out=1)
        dw2 = K.group_xty(h, gdy, order)
        dh = K.scatter2scatter(gdy, w2, order, 1, GROUPED_TO_GROUPED, transpose_w=True, out=h,
                               activation=activation, act_grad_of=h_pre)
        xbar = K.group(r, order, fan_out=1, out=gdy)  # dY_bar is dead after dW2 and dH
        dw1 = K.group_xty(xbar, dh, order)
        dr = K.scatter2scatter(dh, w1, order, 1, GROUPED_TO_SCATTERED, transpose_w=True)
        return dr, dw1, dw2


# ---------------------------------------------------------------------------
# the EP layer

def _a2a(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group):
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


@dataclass
class EpContext:
    x: torch.Tensor
    order: GroupedOrder
    p: torch.Tensor
    k: int
    y_slot: torch.Tensor
    r: torch.Tensor
    saved: tuple
    in_splits: list
    out_splits: list
    activation: str


@dataclass
class EpGradients:
    dx: torch.Tensor
    dw1: torch.Tensor   # local expert slice
    dw2: torch.Tensor
    dp: torch.Tensor


class ExpertParallelSmoeMlp:
    """SMoE MLP with experts sharded over ``group`` (one process per GPU).

    w1_local: (E/G, d_model, d_expert), w2_local: (E/G, d_expert, d_model) — the
    slices of the global expert stacks this rank owns (experts
    [rank*E/G, (rank+1)*E/G)).
    """

    def __init__(self, w1_local, w2_local, num_experts: int, group=None, activation: str = "gelu", ops=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts % self.world:
            raise ValueError(f"num_experts={num_experts} not divisible by world size {self.world}")
        if w1_local.shape[0] != num_experts // self.world or w2_local.shape[0] != num_experts // self.world:
            raise ValueError("local expert slices must hold E/G experts")
        self.w1, self.w2 = w1_local, w2_local
        self.num_experts = num_experts
        self.activation = activation
        self.ops = ops or CudaOps()

    def forward(self, x: torch.Tensor, routing: RoutingResult):
        ops, g = self.ops, self.group
        k = routing.k
        order = ops.order(routing, self.num_experts)
        sc = send_counts(order, self.world)                                   # (G, E_l)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=g)                               # counts exchange
        in_splits = sc.sum(1).tolist()                                        # the one host sync
        out_splits = rc.sum(1).tolist()
        send = ops.group(x, order.o, k)                                       # pack (grouped, rank-major)
        r = torch.empty((sum(out_splits), x.shape[1]), dtype=x.dtype, device=x.device)
        _a2a(r, send, out_splits, in_splits, g)                               # dispatch
        o_loc, off_loc = local_order_from_counts(rc)
        y_recv, saved = ops.local_forward(r, self.w1, self.w2, o_loc, off_loc, self.activation)
        y_back = torch.empty((order.num_slots, x.shape[1]), dtype=x.dtype, device=x.device)
        _a2a(y_back, y_recv, in_splits, out_splits, g)                        # return
        y_slot = ops.group(y_back, order.inverse(), 1)                        # grouped -> slot order
        y = ops.combine(routing.p, y_slot)
        ctx = EpContext(x=x, order=order, p=routing.p, k=k, y_slot=y_slot, r=r, saved=saved,
                        in_splits=in_splits, out_splits=out_splits, activation=self.activation)
        return y, ctx

    def backward(self, ctx: EpContext, dy: torch.Tensor) -> EpGradients:
        ops, g = self.ops, self.group
        t, k = ctx.p.shape
        dp = ops.combine_grad_p(dy, ctx.y_slot, t, k)
        gdy = ops.group(dy, ctx.order.o, k, weights=ctx.p.reshape(-1))       # p-weighted, grouped
        dy_recv = torch.empty((sum(ctx.out_splits), dy.shape[1]), dtype=dy.dtype, device=dy.device)
        _a2a(dy_recv, gdy, ctx.out_splits, ctx.in_splits, g)
        dr, dw1, dw2 = ops.local_backward(ctx.r, self.w1, self.w2, ctx.saved, dy_recv, ctx.activation)
        dx_g = torch.empty((ctx.order.num_slots, dy.shape[1]), dtype=dy.dtype, device=dy.device)
        _a2a(dx_g, dr, ctx.in_splits, ctx.out_splits, g)
        dx_slot = ops.group(dx_g, ctx.order.inverse(), 1)
        dx = ops.fanout_reduce(dx_slot, k)
        return EpGradients(dx=dx, dw1=dw1, dw2=dw2, dp=dp)
