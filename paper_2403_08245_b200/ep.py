"""Expert parallelism (EP) for the SMoE MLP over NCCL: experts sharded over the GPUs of one box.

SURVEY.md §8(e).  The reference has no multi-device code.  Rank r
owns the contiguous expert range [r*E_l, (r+1)*E_l) (E_l = E / G) and its
W1/W2 slices.  This is the NCCL all-to-all-v form (the fallback of the
peer-memory path in ep_peer.py, same sharding and the same routing-weight-
scaled MLP form).  Per forward:

  1. K1 sort of the local routing over the GLOBAL expert ids.
  2. counts all-to-all (G x E_l), the step's one host read (NCCL's split sizes).
  3. pack: the source's rows in (local expert, destination) order —
     send = group(X, o_pack, fan_out=k) with their routing weights — so local
     expert `le`'s rows for every destination are one contiguous chunk.
  4. dispatch chunk by chunk: one all-to-all-v per local expert on a
     communication stream; chunk `le` lands right after chunk `le - 1`, so the
     receive buffer is already in the owner's local grouped order (expert-major,
     then source, then the source's order — the row order of a single GPU on
     the concatenated batch, hence bit-identical results), and the owner's
     layer-1 GEMM of expert `le` starts as soon as its chunk has landed while
     the next chunks are in flight (the tcgen05 GEMMs can leave SMs free for
     NCCL: smoe_set_sm_reserve);
  5. local expert MLP on the received rows in place (grouped in, TMA-fed):
     hp = p * act(x W1) and Y_hat_p = hp W2;
  6. reverse all-to-all-v of Y_hat_p per chunk; the source un-permutes into
     slot order and the combine is the k-sum (p already applied).
Backward mirrors it: the unweighted dY rows go out the same way, the owner's
dH GEMM applies p and produces the dp partials (returned per row, summed at
the source's slot), dW stays local (no all-reduce for expert weights), and the
slot input-gradients come back and are reduced over the k slots.

The local compute and the pack / unpack row ops go through an ``ops`` object.
The default is :class:`CudaOps` (the sm_100a kernels of libsmoe_b200.so); the
CPU multi-process tests inject a torch / NumPy reference to exercise the
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
# index algebra (device-agnostic torch)

def local_order_from_counts(counts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Grouped order of rows received source-major, from the (G sources x E_l experts) counts.

    (Kept for the peer-memory layout tests: ep_peer.dispatch_layout places rows
    directly at these positions.)  Received rows laid out source-major (each
    source's segment in its own expert-major grouped order); the local grouped
    order is expert-major, then source, then the source's order.  Returns
    (o_loc int64 [n_recv], offsets int64 [E_l+1]).
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


def pack_positions(bin_offsets: torch.Tensor, world: int) -> torch.Tensor:
    """Grouped positions in (local expert, destination) order (int64 [n]).

    Global expert q*E_l + le's bin is chunk le's segment for destination q:
    packing the rows in this order makes each local expert's rows for all
    destinations one contiguous all-to-all-v chunk."""
    off = bin_offsets.to(torch.int64)
    e = off.numel() - 1
    el = e // world
    counts = off[1:] - off[:-1]
    ordered = torch.arange(e, device=off.device).view(world, el).t().reshape(-1)   # e = q*el + le, le-major
    lengths = counts[ordered]
    starts = off[:-1][ordered]
    seg = torch.cumsum(lengths, 0) - lengths
    n = int(off[-1])
    within = torch.arange(n, device=off.device) - torch.repeat_interleave(seg, lengths, output_size=n)
    return torch.repeat_interleave(starts, lengths, output_size=n) + within


# ---------------------------------------------------------------------------
# compute backends

class CudaOps:
    """Routing sort, pack / unpack rows and the local expert MLP on the sm_100a kernels."""

    @staticmethod
    def order(routing: RoutingResult, num_experts: int) -> GroupedOrder:
        return compute_grouped_order(routing, num_experts)

    @staticmethod
    def gather(x, rows_o32, fan_out):
        """out[i] = x[rows[i] // fan_out] (group() over an arbitrary row list)."""
        o = GroupedOrder(o=rows_o32, bin_offsets=torch.zeros(2, dtype=torch.int32, device=x.device), validate=False)
        return K.group(x, o, fan_out=fan_out)

    @staticmethod
    def fanout_reduce(g, fan_out):
        return K.fanout_reduce(g, fan_out)

    @staticmethod
    def local_forward(r, p_recv, w1, w2, off_loc, activation, wait=None):
        """Scaled expert MLP on rows in local grouped order: hp = p * act(r W1), y = hp W2.

        Layer 1 runs expert by expert, each launch after wait(le) (its chunk landed),
        so it overlaps the later chunks' all-to-all; tiles never cross experts, so
        the per-expert launches give the same bits as one grouped launch."""
        n, de = r.shape[0], w1.shape[2]
        order = GroupedOrder(o=torch.arange(n, dtype=torch.int32, device=r.device),
                             bin_offsets=off_loc.to(device=r.device, dtype=torch.int32), validate=False)
        h_pre = torch.empty((n, de), dtype=r.dtype, device=r.device)
        hp = torch.empty_like(h_pre)
        offs = [int(v) for v in off_loc.tolist()]
        for le in range(w1.shape[0]):
            a, b = offs[le], offs[le + 1]
            if wait is not None:
                wait(le)
            if b == a:
                continue
            o1 = GroupedOrder(o=order.o[: b - a], bin_offsets=torch.tensor([0, b - a], dtype=torch.int32,
                                                                            device=r.device), validate=False)
            K.scatter2scatter_scaled(r[a:b], w1[le:le + 1], o1, 1, GROUPED_TO_GROUPED, row_scale=p_recv[a:b],
                                     activation=activation, out=h_pre[a:b], act_out=hp[a:b])
        y = K.scatter2scatter(hp, w2, order, 1, GROUPED_TO_GROUPED)
        return y, (order, h_pre, hp)

    @staticmethod
    def local_backward(r, p_recv, w1, w2, saved, dy, activation):
        """dW2 = hp^T dY; dH = p * (dY W2^T) * act'(h_pre) with dp = <dY W2^T, act(h_pre)> per row;
        dW1 = r^T dH; dr = dH W1^T."""
        order, h_pre, hp = saved
        dw2 = K.group_xty(hp, dy, order)
        parts = torch.empty((r.shape[0], K.dp_parts(w1.shape[2])), dtype=torch.float32, device=r.device)
        dh = K.scatter2scatter_scaled(dy, w2, order, 1, GROUPED_TO_GROUPED, row_scale=p_recv, activation=activation,
                                      out=hp, act_grad_of=h_pre, dp_partials=parts, transpose_w=True)
        dp_recv = K.dp_from_partials(parts, order, r.shape[0], 1).view(-1)
        dw1 = K.group_xty(r, dh, order)
        dr = K.scatter2scatter(dh, w1, order, 1, GROUPED_TO_GROUPED, transpose_w=True)
        return dr, dw1, dw2, dp_recv


# ---------------------------------------------------------------------------
# the EP layer

@dataclass
class EpContext:
    order: GroupedOrder
    p: torch.Tensor
    k: int
    pos: torch.Tensor          # slot -> packed position (int32)
    r: torch.Tensor
    p_recv: torch.Tensor
    saved: tuple
    send_chunks: list          # [le][q] rows sent
    recv_chunks: list          # [le][s] rows received
    activation: str


@dataclass
class EpGradients:
    dx: torch.Tensor
    dw1: torch.Tensor   # local expert slice
    dw2: torch.Tensor
    dp: torch.Tensor


class ExpertParallelSmoeMlp:
    """SMoE MLP with experts sharded over ``group`` (one process per GPU), NCCL exchange.

    w1_local: (E/G, d_model, d_expert), w2_local: (E/G, d_expert, d_model) — the
    slices of the global expert stacks this rank owns (experts
    [rank*E/G, (rank+1)*E/G)).  Chunks of the dispatch run on a separate CUDA
    stream when the tensors live on a GPU.
    """

    def __init__(self, w1_local, w2_local, num_experts: int, group=None, activation: str = "gelu", ops=None,
                 sm_reserve: int = 8):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts % self.world:
            raise ValueError(f"num_experts={num_experts} not divisible by world size {self.world}")
        if w1_local.shape[0] != num_experts // self.world or w2_local.shape[0] != num_experts // self.world:
            raise ValueError("local expert slices must hold E/G experts")
        self.w1, self.w2 = w1_local, w2_local
        self.num_experts = num_experts
        self.e_local = num_experts // self.world
        self.activation = activation
        self.ops = ops or CudaOps()
        self.comm = torch.cuda.Stream(device=w1_local.device) if w1_local.is_cuda else None
        if w1_local.is_cuda and self.world > 1:
            # leave SMs to the NCCL chunks that overlap the expert GEMMs
            from . import _lib
            _lib.check(_lib.load().smoe_set_sm_reserve(int(sm_reserve)), "set_sm_reserve")

    # ---- chunked all-to-all-v ------------------------------------------------
    def _exchange(self, inp: torch.Tensor, send_chunks, recv_chunks, inner: int, reverse: bool = False):
        """All-to-all-v chunk by chunk.  Forward: inp packed [le][q] -> out [le][s]
        (local grouped order); reverse: the opposite.  Returns (out, events) where
        events[le] completes when chunk le has landed (None on CPU)."""
        g = self.world
        sc, rc = (recv_chunks, send_chunks) if reverse else (send_chunks, recv_chunks)
        out = torch.empty((sum(sum(c) for c in rc),) + tuple(inp.shape[1:]), dtype=inp.dtype, device=inp.device)
        events = []
        i0 = o0 = 0
        stream = self.comm
        if stream is not None:
            stream.wait_stream(torch.cuda.current_stream(inp.device))
        for le in range(self.e_local):
            ni, no = sum(sc[le]), sum(rc[le])
            if stream is not None:
                with torch.cuda.stream(stream):
                    dist.all_to_all_single(out[o0:o0 + no], inp[i0:i0 + ni], output_split_sizes=rc[le],
                                           input_split_sizes=sc[le], group=self.group)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                inp.record_stream(stream)
                out.record_stream(stream)
                events.append(ev)
            else:
                dist.all_to_all_single(out[o0:o0 + no], inp[i0:i0 + ni], output_split_sizes=rc[le],
                                       input_split_sizes=sc[le], group=self.group)
                events.append(None)
            i0 += ni
            o0 += no
        return out, events

    def _wait_all(self, events) -> None:
        for ev in events:
            if ev is not None:
                torch.cuda.current_stream().wait_event(ev)

    def forward(self, x: torch.Tensor, routing: RoutingResult):
        ops, g, el = self.ops, self.group, self.e_local
        k = routing.k
        order = ops.order(routing, self.num_experts)
        sc = send_counts(order, self.world)                                   # (G, E_l)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=g)                               # counts exchange
        sc_h, rc_h = sc.cpu(), rc.cpu()                                       # the one host read (NCCL splits)
        send_chunks = [[int(sc_h[q, le]) for q in range(self.world)] for le in range(el)]
        recv_chunks = [[int(rc_h[s, le]) for s in range(self.world)] for le in range(el)]
        packed = pack_positions(order.bin_offsets, self.world)               # grouped positions, (le, q) order
        slots = order.o.to(torch.int64)[packed]                                # slot of each packed row
        pos = torch.empty_like(slots)
        pos[slots] = torch.arange(slots.numel(), device=slots.device)
        send = ops.gather(x, slots.to(torch.int32), k)                        # rows in (le, q) order
        p_send = routing.p.reshape(-1).to(torch.float32)[slots].contiguous()
        p_recv, ev_p = self._exchange(p_send, send_chunks, recv_chunks, 1)
        r, ev_x = self._exchange(send, send_chunks, recv_chunks, x.shape[1])
        off_loc = torch.zeros(el + 1, dtype=torch.int64)
        off_loc[1:] = torch.cumsum(torch.tensor([sum(c) for c in recv_chunks], dtype=torch.int64), 0)

        def landed(le):   # chunk le of the rows and of their routing weights is in place
            self._wait_all([ev_p[le], ev_x[le]])

        y_recv, saved = ops.local_forward(r, p_recv, self.w1, self.w2, off_loc, self.activation, wait=landed)
        y_back, ev_y = self._exchange(y_recv, send_chunks, recv_chunks, x.shape[1], reverse=True)
        self._wait_all(ev_y)
        y_slot = ops.gather(y_back, pos.to(torch.int32), 1)                   # packed -> slot order
        y = ops.fanout_reduce(y_slot, k)                                      # p already applied at the owner
        ctx = EpContext(order=order, p=routing.p, k=k, pos=pos.to(torch.int32), r=r, p_recv=p_recv, saved=saved,
                        send_chunks=send_chunks, recv_chunks=recv_chunks, activation=self.activation)
        return y, ctx

    def backward(self, ctx: EpContext, dy: torch.Tensor) -> EpGradients:
        ops = self.ops
        t, k = ctx.p.shape
        slots = torch.empty_like(ctx.pos)
        slots[ctx.pos.long()] = torch.arange(ctx.pos.numel(), dtype=ctx.pos.dtype, device=ctx.pos.device)
        dy_send = ops.gather(dy.contiguous(), slots, k)                       # unweighted dY rows, (le, q) order
        dy_recv, ev = self._exchange(dy_send, ctx.send_chunks, ctx.recv_chunks, dy.shape[1])
        self._wait_all(ev)
        dr, dw1, dw2, dp_recv = ops.local_backward(ctx.r, ctx.p_recv, self.w1, self.w2, ctx.saved, dy_recv,
                                                   ctx.activation)
        dx_back, ev_dx = self._exchange(dr, ctx.send_chunks, ctx.recv_chunks, dy.shape[1], reverse=True)
        dp_back, ev_dp = self._exchange(dp_recv, ctx.send_chunks, ctx.recv_chunks, 1, reverse=True)
        self._wait_all(ev_dx)
        self._wait_all(ev_dp)
        dx_slot = ops.gather(dx_back, ctx.pos, 1)
        dx = ops.fanout_reduce(dx_slot, k)
        dp = dp_back[ctx.pos.long()].view(t, k)
        return EpGradients(dx=dx, dw1=dw1, dw2=dw2, dp=dp)
