"""Expert parallelism over peer memory: dispatch and combine by direct stores.

SURVEY.md §8(e) / §8(f)-2.  Same sharding and row order as ``ep.py`` (rank r
owns experts [r*E_l, (r+1)*E_l); the received rows of a local expert are
ordered by source rank, then by the source's grouped order, so every result
is bit-identical to one GPU running the concatenated batch), but no NCCL
all-to-all and no pack / unpack copies:

  forward   1. each rank zeroes its arrival counters, then a device barrier:
               every peer is done with the previous step's buffers;
            2. each rank stores its per-expert counts (E int64) into row `me`
               of every peer's count table, signal + wait; the receive layout
               (dstart, local bin offsets) is computed from the table ON THE
               DEVICE — no host synchronisation anywhere in the step, which
               therefore captures into a CUDA graph;
            3. dispatch kernel: grouped row i of this rank goes straight to row
               dstart[e] + (i - off[e]) of the owner's receive buffer — its
               final position in the owner's local grouped order — together
               with its slot id, the source rank and its routing weight; experts
               go out in (local expert, owner) order and every 64-row chunk
               bumps the owner's arrival counter of that expert;
            4. the owner runs layer 1 on the received rows as they land: each
               GEMM tile of local expert e waits (in the TMA producer) for
               e's arrival counter, so the dispatch of later experts overlaps
               the first experts' GEMM (grouped in, grouped out, TMA-fed);
            5. layer 2's GEMM epilogue stores output row j straight into row
               slot[j] of its source's slot-ordered buffer (the combine-side
               all-to-all fused into the expert GEMM); the source combines
               with p.
  backward  p-weighted dY rows are dispatched to the same positions; the
            owner's dW2, dH, dW1 and slot input-gradients run on grouped rows
            only (dW stays local: no all-reduce); the input-gradient GEMM's
            epilogue stores the slot gradients into the source's buffer, which
            reduces over the k slots.

Receive buffers hold ``capacity`` rows: by default the exact worst case (every
rank's rows on one owner, G*T*k), or ceil(capacity_factor * T * k) rows.  A
step whose routing sends more rows to a rank than it can hold does not write
past the buffer: the overflow bit of the device error word is set and
``check()`` raises (``check()`` is the only host read; call it when a step's
results are consumed, e.g. at logging intervals).

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
                 activation: str = "gelu", timeout_s: float = 60.0, scaled: bool | None = None,
                 capacity_factor: float | None = None):
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
        self.e_local = el
        self.max_tokens = max_tokens
        self.timeout_ns = int(timeout_s * 1e9)
        # the routing weight travels with the row and moves through layer 2 at
        # the owner (moe_layers.py's scaled form): the source's combine becomes
        # a k-sum and dp comes back from the owner's dH epilogue
        from . import moe_layers
        self.scaled = moe_layers._SCALED if scaled is None else bool(scaled)
        dev = w1_local.device
        d = w1_local.shape[1]
        de = w1_local.shape[2]
        self.d = d
        g = self.world
        slots = max_tokens * k
        worst = slots * g                                # every rank's rows on one owner
        if capacity_factor is None:
            cap = worst
        else:
            if capacity_factor <= 0:
                raise ValueError(f"capacity_factor must be > 0, got {capacity_factor}")
            cap = min(worst, -(-int(capacity_factor * slots) // 256) * 256)
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
        # arrival counters of the forward (x rows) and backward (dY rows) dispatch, E_l each
        self.arrive = SymmetricBuffer(8 * 2 * el, dev, group)
        self.arrive_bwd_peers = self.arrive.peers + 8 * el
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.my_epochs = torch.zeros(_NUM_SLOTS, dtype=torch.int64, device=dev)
        # persistent per-step buffers (no allocation inside the step)
        self.h_pre = torch.empty((cap, de), dtype=torch.bfloat16, device=dev)
        self.h = torch.empty_like(self.h_pre)
        self.parts = torch.empty((cap, K.dp_parts(de)), dtype=torch.float32, device=dev) if self.scaled else None
        self.o_loc = torch.arange(cap, dtype=torch.int32, device=dev)
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
        """Signal every peer for `slot`, then wait for every peer's signal (device-side epochs)."""
        lib = _lib.load()
        t0 = _lt.begin()
        _lib.check(lib.smoe_ep_signal(self.flags.peers.data_ptr(), self.world, self.rank, slot,
                                      self.my_epochs.data_ptr(), _stream()), "ep_signal")
        _lib.check(lib.smoe_ep_wait(self.flags.local.data_ptr(), self.world, slot, self.my_epochs.data_ptr(),
                                    self.timeout_ns, self.err.data_ptr(), _stream()), "ep_wait")
        _lt.end(f"ep_sync {_SLOT_NAMES[slot]}", t0)

    def check(self) -> None:
        """Raise if a step since the last check timed out waiting for a peer or overflowed
        the receive capacity (the one host read of the layer; results of such a step are invalid)."""
        code = int(self.err.item())
        if code:
            self.err.zero_()
            why = []
            if code & 1:
                why.append("a peer did not signal within the timeout")
            if code & 2:
                why.append(f"more rows were routed to a rank than its receive capacity ({self.cap} rows); "
                           f"raise capacity_factor (None = the exact worst case)")
            raise RuntimeError("peer-memory EP: " + "; ".join(why))

    _check_err = check

    # ---- forward / backward ------------------------------------------------------
    def forward(self, x: torch.Tensor, routing: RoutingResult):
        lib = _lib.load()
        k, g, e = routing.k, self.world, self.num_experts
        el = self.e_local
        t = x.shape[0]
        if k != self.k or t > self.max_tokens:
            raise ValueError(f"routing k={k} / {t} tokens exceed the buffers (k={self.k}, max_tokens={self.max_tokens})")
        if x.dtype != torch.bfloat16 or x.shape[1] != self.d:
            raise ValueError("x must be bf16 with d_model columns")
        x = x.contiguous()
        order = compute_grouped_order(routing, e)
        n = order.num_slots
        # 1. this rank's arrival counters start from zero; then every peer is
        #    done with the previous step's buffers (and has zeroed its counters)
        self.arrive.local.zero_()
        self._exchange_done(_READY)
        # 2. count table -> receive layout, on the device
        cnt = order.bin_counts.to(torch.int64).contiguous()
        _call("ep_put counts", lib.smoe_ep_put, cnt.data_ptr(), 8 * e, self.counts.peers.data_ptr(),
              8 * e * self.rank, g, _stream())
        self._exchange_done(_COUNTS)
        table = self.counts.view(torch.int64, (g, e))
        dstart, off_loc = dispatch_layout(table, self.rank)
        off32 = off_loc.clamp(max=self.cap).to(torch.int32)     # never past the receive buffer
        _call("ep_check_capacity", lib.smoe_ep_check_capacity, off_loc.to(torch.int32).data_ptr(), el, self.cap,
              self.err.data_ptr(), _stream())
        order_loc = GroupedOrder(o=self.o_loc, bin_offsets=off32, validate=False)
        # 3. dispatch rows (+ slot ids, source rank, routing weight) to their owners
        pw = routing.p.reshape(-1).to(torch.float32).contiguous()
        self._dispatch(x, order, k, None, dstart, self.recv_x, with_meta=True, pw=pw,
                       arrive=self.arrive.peers if self.scaled else None, label="ep_dispatch x")
        de = self.w1.shape[2]
        r = self.recv_x.view(torch.bfloat16, (self.cap, self.d))
        h_pre, h = self.h_pre, self.h
        if self.scaled:
            # 4. h = p * act(h_pre) on the rows as they land: tiles gated on the arrival counters
            _call("ep_expert_gemm_gated (layer 1)", lib.smoe_ep_expert_gemm_gated,
                  r.data_ptr(), self.cap, self.w1.data_ptr(), el, self.w1.shape[1], de, self.o_loc.data_ptr(),
                  off32.data_ptr(), 0,
                  _lib.EPI_ACT_SCALED, _lib.ACTIVATION_IDS[self.activation], self._recv_p().data_ptr(),
                  h_pre.data_ptr(), h.data_ptr(), None, None, 0, self.arrive.local.data_ptr(), _stream())
        else:
            self._exchange_done(_FWD_DISPATCH)
            K.scatter2scatter(r, self.w1, order_loc, 1, GROUPED_TO_GROUPED, out=h_pre, activation=self.activation,
                              act_out=h)
        # 5. layer 2, its outputs stored back into their source slots; then the
        #    routing-weighted combine at the source
        self._gemm_return(h, self.w2, order_loc, False, self.y_ret)
        self._exchange_done(_FWD_RETURN)
        y_slot = self.y_ret.view(torch.bfloat16, (self.max_tokens * k, self.d))[:n]
        y = K.fanout_reduce(y_slot, k) if self.scaled else K.combine(routing.p, y_slot)
        ctx = PeerEpContext(order=order, p=routing.p, k=k, dstart=dstart, order_loc=order_loc,
                            h_pre=h_pre, h=h, y_slot=y_slot, activation=self.activation)
        return y, ctx

    def backward(self, ctx: PeerEpContext, dy: torch.Tensor) -> PeerEpGradients:
        lib = _lib.load()
        g, e, k = self.world, self.num_experts, ctx.k
        el = self.e_local
        t = ctx.p.shape[0]
        dy = dy.contiguous()
        n = ctx.order.num_slots
        dp = None if self.scaled else K.combine_grad_p(dy, ctx.y_slot, t, k)
        pw = ctx.p.reshape(-1).to(torch.float32).contiguous()
        ol = ctx.order_loc
        off32 = ol.bin_offsets
        # scaled form: unweighted dY rows (p is applied in the owner's dH epilogue)
        self._dispatch(dy, ctx.order, k, None if self.scaled else pw, ctx.dstart, self.recv_dy, with_meta=False,
                       arrive=self.arrive_bwd_peers if self.scaled else None, label="ep_dispatch dy")
        dyl = self.recv_dy.view(torch.bfloat16, (self.cap, self.d))
        r = self.recv_x.view(torch.bfloat16, (self.cap, self.d))
        de = self.w1.shape[2]
        if self.scaled:
            arrive_bwd = self.arrive.local.data_ptr() + 8 * el
            # dW2 = hp^T dY and dH = p * (dY W2^T) * act'(h_pre) (+ dp partials), each
            # tile gated on the arrival of its expert's dY rows
            dw2 = torch.empty((el, de, self.d), dtype=torch.bfloat16, device=dy.device)
            _call("ep_group_xty_gated (dW2)", lib.smoe_ep_group_xty_gated, ctx.h.data_ptr(), dyl.data_ptr(),
                  off32.data_ptr(), el, self.cap, de, self.d, dw2.data_ptr(), arrive_bwd, _stream())
            parts = self.parts
            _call("ep_expert_gemm_gated (dH)", lib.smoe_ep_expert_gemm_gated,
                  dyl.data_ptr(), self.cap, self.w2.data_ptr(), el, de, self.d, self.o_loc.data_ptr(),
                  off32.data_ptr(), 1,
                  _lib.EPI_ACT_GRAD_SCALED, _lib.ACTIVATION_IDS[ctx.activation], self._recv_p().data_ptr(),
                  ctx.h.data_ptr(), None, ctx.h_pre.data_ptr(), parts.data_ptr(), parts.shape[1], arrive_bwd,
                  _stream())
            dh = ctx.h
            _call("ep_dp_return", lib.smoe_ep_dp_return, parts.data_ptr(), self.cap, parts.shape[1],
                  self.recv_slot.local.data_ptr(), self.recv_src.local.data_ptr(), self.dp_ret.peers.data_ptr(),
                  off32[el:].data_ptr(), _stream())
        else:
            self._exchange_done(_BWD_DISPATCH)
            dw2 = K.group_xty(ctx.h, dyl, ol)
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

    def _dispatch(self, src: torch.Tensor, order: GroupedOrder, k: int, weights, dstart, dest: SymmetricBuffer,
                  with_meta: bool, label: str, pw=None, arrive=None) -> None:
        lib = _lib.load()
        _call(label, lib.smoe_ep_dispatch_rows,
              src.data_ptr(), src.shape[0], self.d, order.o.data_ptr(), order.bin_offsets.data_ptr(),
              self.num_experts, k, None if weights is None else weights.data_ptr(), order.num_slots,
              dstart.data_ptr(), self.e_local, self.world, dest.peers.data_ptr(),
              self.recv_slot.peers.data_ptr() if with_meta else None,
              self.recv_src.peers.data_ptr() if with_meta else None, self.rank,
              pw.data_ptr() if (with_meta and self.scaled) else None,
              self.recv_p.peers.data_ptr() if (with_meta and self.scaled) else None, self.cap,
              None if arrive is None else arrive.data_ptr(), self.err.data_ptr(), _lib.SMOE_BF16, _stream())

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
              dest.peers.data_ptr(), order_loc.bin_offsets[self.e_local:].data_ptr(), _lib.SMOE_BF16, _stream())

    def _recv_p(self) -> torch.Tensor:
        return self.recv_p.view(torch.float32, (self.cap,))

    def _buffers(self):
        return (self.flags, self.counts, self.recv_x, self.recv_dy, self.recv_slot, self.recv_src, self.y_ret,
                self.dx_ret, self.recv_p, self.dp_ret, self.arrive)

    def close(self) -> None:
        torch.cuda.synchronize()
        for b in self._buffers():
            b.close()
