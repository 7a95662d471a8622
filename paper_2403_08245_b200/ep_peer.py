"""Expert parallelism over peer memory: dispatch and combine by direct stores.

SURVEY.md §8(e) / §8(f)-2.  Same sharding and row order as ``ep.py`` (rank r
owns experts [r*E_l, (r+1)*E_l); the received rows of a local expert are
ordered by source rank, then by the source's grouped order, so every result
is bit-identical to one GPU running the concatenated batch), but no NCCL
all-to-all and no pack / unpack copies:

  forward   1. device barrier: every peer is done with the previous step's
               buffers;
            2. each rank stores its per-expert counts (E int64) into row `me`
               of every peer's count table, signal + wait; one host read of the
               table gives the receive sizes (the step's only host sync);
            3. dispatch kernel: grouped row i of this rank goes straight to row
               dstart[e] + (i - off[e]) of the owner's receive buffer — its
               final position in the owner's local grouped order — together
               with its slot id and the source rank;
            4. the owner runs layer 1 on the received rows as they landed
               (grouped in, grouped out: TMA-fed, no group() copy);
            5. layer 2's GEMM epilogue stores output row j straight into row
               slot[j] of its source's slot-ordered buffer (the combine-side
               all-to-all fused into the expert GEMM); the source combines
               with p.
  backward  p-weighted dY rows are dispatched to the same positions; the
            owner's dW2, dH, dW1 and slot input-gradients run on grouped rows
            only (dW stays local: no all-reduce); the input-gradient GEMM's
            epilogue stores the slot gradients into the source's buffer, which
            reduces over the k slots.

Peer buffers are CUDA IPC mappings of each rank's buffers (``SymmetricBuffer``);
the store kernels write through NVLink P2P on a multi-GPU box and into the
same device's memory when the ranks share one GPU (the test rig).  Completion
is signalled with system-scope fences and per-source flag counters; a wait
that exceeds ``timeout_s`` raises instead of hanging the device.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from . import kernels as K
from . import launch_timer as _lt
from .kernels import GROUPED_TO_GROUPED
from .router import GroupedOrder, RoutingResult, compute_grouped_order

# flag slots: one counter per (slot, source rank) on every rank
_READY, _COUNTS, _FWD_DISPATCH, _FWD_RETURN, _BWD_DISPATCH, _BWD_RETURN = range(6)
_NUM_SLOTS = 6

# The return is fused into the expert GEMM (its epilogue stores each output row
# into the source's buffer); SMOE_EP_FUSED_RETURN=0 runs GEMM + return kernel.
_FUSED_RETURN = os.environ.get("SMOE_EP_FUSED_RETURN", "1") != "0"


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _call(label: str, fn, *args) -> None:
    """One C-ABI call, timed under `label` when a LaunchTimer is active."""
    t0 = _lt.begin()
    st = fn(*args)
    _lt.end(label, t0)
    _lib.check(st, label)


_SLOT_NAMES = ("ready", "counts", "fwd dispatch", "fwd return", "bwd dispatch", "bwd return")


class SymmetricBuffer:
    """One device buffer per rank, every rank's copy addressable by every rank.

    ``peers`` is a device int64 tensor of the world's base addresses (this
    rank's own buffer at index ``rank``), the table the store kernels index.
    """

    def __init__(self, nbytes: int, device: torch.device, group=None):
        lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local = torch.zeros(max(int(nbytes), 16), dtype=torch.uint8, device=device)
        handle = ctypes.create_string_buffer(lib.smoe_ipc_handle_bytes())
        offset = ctypes.c_int64()
        _lib.check(lib.smoe_ipc_get_handle(self.local.data_ptr(), handle, ctypes.byref(offset)), "ipc_get_handle")
        torch.cuda.synchronize(device)    # zero-fill visible before peers map it
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (handle.raw, offset.value), group=group)
        self._opened: list[int] = []
        self.error: str | None = None     # a failed mapping is reported collectively by the owner
        ptrs = []
        for q, (raw, off) in enumerate(gathered):
            if q == self.rank:
                ptrs.append(self.local.data_ptr())
                continue
            base = ctypes.c_void_p()
            if lib.smoe_ipc_open(raw, ctypes.byref(base)) != 0:
                self.error = f"rank {self.rank}: cannot map rank {q}'s buffer: {_lib.last_error()}"
                ptrs.append(0)
                continue
            self._opened.append(base.value)
            ptrs.append(base.value + off)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)

    def view(self, dtype: torch.dtype, shape) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= int(s)
        return self.local[: n * torch.empty((), dtype=dtype).element_size()].view(dtype).view(*shape)

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.smoe_ipc_close(ctypes.c_void_p(p))
        self._opened = []


@dataclass
class PeerEpContext:
    order: GroupedOrder
    p: torch.Tensor
    k: int
    dstart: torch.Tensor
    n_recv: int
    order_loc: GroupedOrder
    h_pre: torch.Tensor
    h: torch.Tensor
    y_slot: torch.Tensor
    activation: str


@dataclass
class PeerEpGradients:
    dx: torch.Tensor
    dw1: torch.Tensor
    dw2: torch.Tensor
    dp: torch.Tensor


def dispatch_layout(counts: torch.Tensor, me: int) -> tuple[torch.Tensor, torch.Tensor]:
    """From the (G sources x E global experts) count table: this source's first
    receive row per global expert at its owner (dstart, int64 [E]) and this
    rank's local bin offsets (int64 [E_l + 1]).

    Owner q's receive buffer is expert-major over its experts, then source-major
    inside each expert — the grouped order of the concatenated batch."""
    g, e = counts.shape
    el = e // g
    c = counts.to(torch.int64)
    tot = c.sum(0).view(g, el)                                   # rows per (owner, local expert)
    start_of_expert = (torch.cumsum(tot, 1) - tot).reshape(e)    # local bin start at the owner
    below = torch.cumsum(c, 0) - c                               # rows from lower source ranks
    dstart = start_of_expert + below[me]
    off_loc = torch.zeros(el + 1, dtype=torch.int64, device=counts.device)
    off_loc[1:] = torch.cumsum(tot[me], 0)
    return dstart, off_loc


class PeerExpertParallelSmoeMlp:
    """SMoE MLP with experts sharded over ``group``, exchanging rows through peer memory.

    w1_local (E/G, d_model, d_expert) and w2_local (E/G, d_expert, d_model) are
    this rank's expert slices.  ``max_tokens`` bounds the tokens per rank and
    call (buffers are sized for the worst case: every routed row of every rank
    landing on one owner).
    """

    def __init__(self, w1_local, w2_local, num_experts: int, k: int, max_tokens: int, group=None,
                 activation: str = "gelu", timeout_s: float = 60.0, scaled: bool | None = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts % self.world:
            raise ValueError(f"num_experts={num_experts} not divisible by world size {self.world}")
        el = num_experts // self.world
        if w1_local.shape[0] != el or w2_local.shape[0] != el:
            raise ValueError("local expert slices must hold E/G experts")
        if w1_local.dtype != torch.bfloat16:
            raise ValueError("the peer-memory EP path runs the bf16 tensor-core kernels")
        self.w1, self.w2 = w1_local, w2_local
        self.num_experts, self.k, self.activation = num_experts, k, activation
        self.max_tokens = max_tokens
        self.timeout_ns = int(timeout_s * 1e9)
        # the routing weight travels with the row and moves through layer 2 at
        # the owner (moe_layers.py's scaled form): the source's combine becomes
        # a k-sum and dp comes back from the owner's dH epilogue
        from . import moe_layers
        self.scaled = moe_layers._SCALED if scaled is None else bool(scaled)
        dev = w1_local.device
        d = w1_local.shape[1]
        self.d = d
        g = self.world
        slots = max_tokens * k
        cap = slots * g                                  # worst case: all rows to one owner
        self.cap = cap
        esz = 2
        self.flags = SymmetricBuffer(8 * _NUM_SLOTS * g, dev, group)
        self.counts = SymmetricBuffer(8 * g * num_experts, dev, group)
        self.recv_x = SymmetricBuffer(esz * cap * d, dev, group)
        self.recv_dy = SymmetricBuffer(esz * cap * d, dev, group)
        self.recv_slot = SymmetricBuffer(4 * cap, dev, group)
        self.recv_src = SymmetricBuffer(4 * cap, dev, group)
        self.y_ret = SymmetricBuffer(esz * slots * d, dev, group)
        self.dx_ret = SymmetricBuffer(esz * slots * d, dev, group)
        self.recv_p = SymmetricBuffer(4 * cap, dev, group)      # routing weight of each received row
        self.dp_ret = SymmetricBuffer(4 * slots, dev, group)    # dp per slot, returned by the owners
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = [0] * _NUM_SLOTS
        # every rank must have mapped every peer buffer; decide collectively so
        # all ranks raise together (a caller can then fall back to ep.py)
        errors = [b.error for b in self._buffers() if b.error]
        gathered = [None] * g
        dist.all_gather_object(gathered, errors[0] if errors else None, group=group)
        bad = [e for e in gathered if e]
        if bad:
            self.close()
            raise RuntimeError("peer-memory EP unavailable: " + "; ".join(bad))

    # ---- completion ------------------------------------------------------------
    def _exchange_done(self, slot: int) -> None:
        """Signal every peer for `slot`, then wait for every peer's signal."""
        lib = _lib.load()
        self.epoch[slot] += 1
        t0 = _lt.begin()
        _lib.check(lib.smoe_ep_signal(self.flags.peers.data_ptr(), self.world, self.rank, slot, _stream()),
                   "ep_signal")
        _lib.check(lib.smoe_ep_wait(self.flags.local.data_ptr(), self.world, slot, self.epoch[slot],
                                    self.timeout_ns, self.err.data_ptr(), _stream()), "ep_wait")
        _lt.end(f"ep_sync {_SLOT_NAMES[slot]}", t0)

    def _check_err(self) -> None:
        if int(self.err.item()):
            raise RuntimeError("peer-memory EP: a peer did not signal within the timeout")

    # ---- forward / backward ------------------------------------------------------
    def forward(self, x: torch.Tensor, routing: RoutingResult):
        lib = _lib.load()
        k, g, e = routing.k, self.world, self.num_experts
        t = x.shape[0]
        if k != self.k or t > self.max_tokens:
            raise ValueError(f"routing k={k} / {t} tokens exceed the buffers (k={self.k}, max_tokens={self.max_tokens})")
        if x.dtype != torch.bfloat16 or x.shape[1] != self.d:
            raise ValueError("x must be bf16 with d_model columns")
        x = x.contiguous()
        order = compute_grouped_order(routing, e)
        n = order.num_slots
        # 1. previous step's buffers are free everywhere
        self._exchange_done(_READY)
        # 2. count table
        cnt = order.bin_counts.to(torch.int64).contiguous()
        _call("ep_put counts", lib.smoe_ep_put, cnt.data_ptr(), 8 * e, self.counts.peers.data_ptr(),
              8 * e * self.rank, g, _stream())
        self._exchange_done(_COUNTS)
        table = self.counts.view(torch.int64, (g, e))
        dstart, off_loc = dispatch_layout(table, self.rank)
        n_recv = int(off_loc[-1])                      # the one host sync of the step
        self._check_err()
        # 3. dispatch rows (+ slot ids, source rank, routing weight) to their owners
        pw = routing.p.reshape(-1).to(torch.float32).contiguous()
        _call("ep_dispatch x", lib.smoe_ep_dispatch_rows,
              x.data_ptr(), t, self.d, order.o.data_ptr(), order.sorted_expert_idxs.data_ptr(),
              order.bin_offsets.data_ptr(), k, None, n, dstart.data_ptr(), e // g, self.recv_x.peers.data_ptr(),
              self.recv_slot.peers.data_ptr(), self.recv_src.peers.data_ptr(), self.rank,
              pw.data_ptr() if self.scaled else None, self.recv_p.peers.data_ptr() if self.scaled else None,
              _lib.SMOE_BF16, _stream())
        self._exchange_done(_FWD_DISPATCH)
        # 4. local experts on the landed rows (grouped in, grouped out)
        r = self.recv_x.view(torch.bfloat16, (self.cap, self.d))[:n_recv]
        order_loc = GroupedOrder(o=torch.arange(n_recv, dtype=torch.int32, device=x.device),
                                 bin_offsets=off_loc.to(torch.int32), validate=False)
        de = self.w1.shape[2]
        h_pre = torch.empty((n_recv, de), dtype=x.dtype, device=x.device)
        h = torch.empty_like(h_pre)
        if self.scaled:   # h = p * act(h_pre); order_loc is the identity, so row i's scale is recv_p[i]
            K.scatter2scatter_scaled(r, self.w1, order_loc, 1, GROUPED_TO_GROUPED, row_scale=self._recv_p(n_recv),
                                     activation=self.activation, out=h_pre, act_out=h)
        else:
            K.scatter2scatter(r, self.w1, order_loc, 1, GROUPED_TO_GROUPED, out=h_pre, activation=self.activation,
                              act_out=h)
        # 5. layer 2, its outputs stored back into their source slots; then the
        #    routing-weighted combine at the source
        self._gemm_return(h, self.w2, order_loc, False, self.y_ret)
        self._exchange_done(_FWD_RETURN)
        y_slot = self.y_ret.view(torch.bfloat16, (self.max_tokens * k, self.d))[:n]
        y = K.fanout_reduce(y_slot, k) if self.scaled else K.combine(routing.p, y_slot)
        ctx = PeerEpContext(order=order, p=routing.p, k=k, dstart=dstart, n_recv=n_recv, order_loc=order_loc,
                            h_pre=h_pre, h=h, y_slot=y_slot, activation=self.activation)
        return y, ctx

    def backward(self, ctx: PeerEpContext, dy: torch.Tensor) -> PeerEpGradients:
        lib = _lib.load()
        g, e, k = self.world, self.num_experts, ctx.k
        t = ctx.p.shape[0]
        dy = dy.contiguous()
        n = ctx.order.num_slots
        dp = None if self.scaled else K.combine_grad_p(dy, ctx.y_slot, t, k)
        pw = ctx.p.reshape(-1).to(torch.float32).contiguous()
        # scaled form: unweighted dY rows (p is applied in the owner's dH epilogue)
        _call("ep_dispatch dy", lib.smoe_ep_dispatch_rows,
              dy.data_ptr(), t, self.d, ctx.order.o.data_ptr(), ctx.order.sorted_expert_idxs.data_ptr(),
              ctx.order.bin_offsets.data_ptr(), k, None if self.scaled else pw.data_ptr(), n, ctx.dstart.data_ptr(),
              e // g, self.recv_dy.peers.data_ptr(), None, None, self.rank, None, None, _lib.SMOE_BF16, _stream())
        self._exchange_done(_BWD_DISPATCH)
        nr = ctx.n_recv
        dyl = self.recv_dy.view(torch.bfloat16, (self.cap, self.d))[:nr]
        r = self.recv_x.view(torch.bfloat16, (self.cap, self.d))[:nr]
        ol = ctx.order_loc
        dw2 = K.group_xty(ctx.h, dyl, ol)
        if self.scaled:   # dH = p * (dY W2^T) * act'(h_pre), dp partials from the same accumulators
            parts = torch.empty((nr, K.dp_parts(self.w1.shape[2])), dtype=torch.float32, device=dy.device)
            dh = K.scatter2scatter_scaled(dyl, self.w2, ol, 1, GROUPED_TO_GROUPED, row_scale=self._recv_p(nr),
                                          activation=ctx.activation, out=ctx.h, act_grad_of=ctx.h_pre,
                                          dp_partials=parts, transpose_w=True)
            _call("ep_dp_return", lib.smoe_ep_dp_return, parts.data_ptr(), nr, parts.shape[1],
                  self.recv_slot.local.data_ptr(), self.recv_src.local.data_ptr(), self.dp_ret.peers.data_ptr(),
                  _stream())
        else:
            dh = K.scatter2scatter(dyl, self.w2, ol, 1, GROUPED_TO_GROUPED, transpose_w=True, out=ctx.h,
                                   activation=ctx.activation, act_grad_of=ctx.h_pre)
        dw1 = K.group_xty(r, dh, ol)
        self._gemm_return(dh, self.w1, ol, True, self.dx_ret, scratch=dyl)
        self._exchange_done(_BWD_RETURN)
        dx_slot = self.dx_ret.view(torch.bfloat16, (self.max_tokens * k, self.d))[:n]
        dx = K.fanout_reduce(dx_slot, k)
        if self.scaled:
            dp = self.dp_ret.view(torch.float32, (self.max_tokens * k,))[:n].reshape(t, k).clone()
        return PeerEpGradients(dx=dx, dw1=dw1, dw2=dw2, dp=dp)

    def _gemm_return(self, a: torch.Tensor, w: torch.Tensor, order_loc: GroupedOrder, transpose: bool,
                     dest: SymmetricBuffer, scratch: torch.Tensor | None = None) -> None:
        """rows a @ W[e] (W[e]^T) of the local grouped order, each stored into its
        source's slot row of `dest` — in the GEMM epilogue when fused."""
        lib = _lib.load()
        n = a.shape[0]
        slot, src = self.recv_slot.local.data_ptr(), self.recv_src.local.data_ptr()
        if _FUSED_RETURN:
            _call("ep_gemm_return " + ("W^T (dX)" if transpose else "(layer 2)"), lib.smoe_ep_gemm_return,
                  a.data_ptr(), n, w.data_ptr(), w.shape[0], w.shape[1], w.shape[2], order_loc.bin_offsets.data_ptr(),
                  int(transpose), slot, src, dest.peers.data_ptr(), _stream())
            return
        out = K.scatter2scatter(a, w, order_loc, 1, GROUPED_TO_GROUPED, transpose_w=transpose, out=scratch)
        _call("ep_return rows", lib.smoe_ep_return_rows, out.data_ptr(), n, self.d, slot, src,
              dest.peers.data_ptr(), _lib.SMOE_BF16, _stream())

    def _recv_p(self, rows: int) -> torch.Tensor:
        return self.recv_p.view(torch.float32, (self.cap,))[:rows]

    def _buffers(self):
        return (self.flags, self.counts, self.recv_x, self.recv_dy, self.recv_slot, self.recv_src, self.y_ret,
                self.dx_ret, self.recv_p, self.dp_ret)

    def close(self) -> None:
        torch.cuda.synchronize()
        for b in self._buffers():
            b.close()
