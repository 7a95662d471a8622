"""scattermlp-compatible wrappers over the C-ABI kernels (fp32 / fp64 check mode).

The reference package (``scattermlp``, /root/reference/pkg/src/scattermlp)
passes NumPy-backed ``Matrix`` / ``ExpertTensor`` / ``GroupedOrder`` objects
between its kernels.  This module accepts exactly those objects, moves them to
the GPU, runs the hot-path kernels of libsmoe_b200.so (fp32 or fp64 storage,
64-bit accumulation, one rounding — the reference's numeric contract,
core_tensor.py:1-7) and hands back objects of the reference's own types, so the
reference's own test suite can run unchanged against the GPU path:

    import scattermlp
    from paper_2403_08245_b200 import refshim
    refshim.install(scattermlp)   # rebinds the hot-path names

What ``install`` rebinds (each one replaces the reference function at
file:line, under /root/reference/pkg/src/scattermlp/):

* ``scatter2scatter`` (kernels.py:143-220), ``scatter_combine`` (:242-286),
  ``group`` (:289-326), ``group_xty`` (:329-361), ``set_fault_injection``
  (:100-107) — in ``scattermlp``, ``scattermlp.kernels`` and
  ``scattermlp.parallel_linear`` (which bound them with ``from .kernels
  import``);
* ``compute_grouped_order`` (router.py:154-164) in the top-level namespace
  (the K1 sort kernel; the oracle's own lazy imports keep NumPy's argsort);
* ``parallel_linear._combine`` (parallel_linear.py:69-73) — the combine row
  kernel;
* ``moe_layers.apply_activation`` / ``activation_grad`` (moe_layers.py:75-83)
  as used by the routed MLP — the activation kernel.

The reference's orchestration (parallel_linear.forward/backward,
smoe_mlp_forward/backward, momha_forward/backward, the ledger) stays its own
code and now drives the GPU kernels, including on the float64 matrices of the
reference's finite-difference gradient checks (SMOE_F64 storage).

Exceptions keep the reference's classes: shape errors surface as the
reference's ``DimensionError``, argument errors as ``ValueError``.
"""
from __future__ import annotations

import contextlib
import weakref

import numpy as np
import torch

from . import kernels as _k
from .errors import DimensionError as _OurDimensionError
from .router import GroupedOrder as _DevOrder
from .router import _sort_ids

_DEVICE = "cuda"


class _Shim:
    def __init__(self, ref):
        import importlib

        self.ref = ref
        self.core = importlib.import_module(ref.__name__ + ".core_tensor")
        self.errors = importlib.import_module(ref.__name__ + ".errors")
        self.kernels = importlib.import_module(ref.__name__ + ".kernels")
        self.router = importlib.import_module(ref.__name__ + ".router")
        self.pl = importlib.import_module(ref.__name__ + ".parallel_linear")
        self.layers = importlib.import_module(ref.__name__ + ".moe_layers")
        self._orders: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()

    # ---- conversions -------------------------------------------------------
    @contextlib.contextmanager
    def _ref_errors(self):
        """Re-raise this package's DimensionError as the reference's class."""
        try:
            yield
        except _OurDimensionError as exc:
            raise self.errors.DimensionError(str(exc)) from None

    @staticmethod
    def _check_dtype(arr: np.ndarray, what: str) -> None:
        if arr.dtype not in (np.float32, np.float64):
            raise ValueError(f"{what}: unsupported element type {arr.dtype}; use float32 or float64")

    def _dev(self, m, what: str) -> torch.Tensor:
        arr = m if isinstance(m, np.ndarray) else m.data   # Matrix / ExpertTensor hold .data
        self._check_dtype(arr, what)
        return torch.from_numpy(np.ascontiguousarray(arr)).to(_DEVICE)

    def _order(self, order) -> _DevOrder:
        dev = self._orders.get(order)
        if dev is None:
            o = torch.from_numpy(np.ascontiguousarray(order.o, dtype=np.int32)).to(_DEVICE)
            off = torch.from_numpy(np.ascontiguousarray(order.bin_offsets, dtype=np.int32)).to(_DEVICE)
            inv = torch.empty_like(o)
            inv[o.long()] = torch.arange(o.numel(), dtype=torch.int32, device=_DEVICE)
            dev = _DevOrder(o=o, bin_offsets=off, inv=inv, validate=False)
            self._orders[order] = dev
        return dev

    def _credit(self, order, d_in: int, d_out: int) -> None:
        # the reference's own counter (kernels.py:74-98): sum_e count_e * d_in * d_out
        self.kernels.add_macs(int(np.sum(order.bin_counts * (d_in * d_out))))

    @staticmethod
    def _host(t: torch.Tensor) -> np.ndarray:
        return t.cpu().numpy()

    def _into(self, out, result: torch.Tensor):
        if out is None:
            return self.core.Matrix(self._host(result))
        out.data[...] = self._host(result)
        return out

    # ---- the reference's kernel API ------------------------------------------
    def scatter2scatter(self, x, w, order, fan_out, layout=None, tile=None, *, transpose_w=False, out=None):
        layout = layout if layout is not None else self.kernels.SCATTERED_TO_SCATTERED
        if fan_out < 1:
            raise ValueError(f"fan_out must be >= 1, got {fan_out}")
        num_slots = order.num_slots
        self.errors.require_dims(order.num_experts == w.num_experts, "order bins vs expert stack",
                                 (order.num_experts,), (w.num_experts,))
        d_in = w.d_out if transpose_w else w.d_in
        d_out = w.d_in if transpose_w else w.d_out
        self.errors.require_dims(x.cols == d_in, "input width vs expert weights", (x.rows, x.cols), (d_in, d_out))
        if layout.grouped_in:
            self.errors.require_dims(x.rows == num_slots, "grouped input rows vs slots", (x.rows,), (num_slots,))
        elif x.rows * fan_out != num_slots:
            raise ValueError(f"scattered input rows ({x.rows}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
        if out is not None:
            self.errors.require_dims(out.rows == num_slots and out.cols == d_out, "out buffer",
                                     (out.rows, out.cols), (num_slots, d_out))
            if out.dtype != x.dtype:
                raise ValueError(f"out dtype {out.dtype} does not match input dtype {x.dtype}")
        with self._ref_errors():
            res = _k.scatter2scatter(self._dev(x, "scatter2scatter x"), self._dev(w, "scatter2scatter w"),
                                     self._order(order), fan_out, layout, transpose_w=transpose_w)
        self._credit(order, d_in, d_out)
        return self._into(out, res)

    def scatter_combine(self, x, w, order, fan_out, p_flat, combine_cols, grouped_in, tile=None):
        if fan_out < 1:
            raise ValueError(f"fan_out must be >= 1, got {fan_out}")
        num_slots = order.num_slots
        if num_slots % combine_cols:
            raise ValueError(f"combine width {combine_cols} must divide T*k ({num_slots})")
        self.errors.require_dims(p_flat.shape == (num_slots,), "combine weights", p_flat.shape, (num_slots,))
        d_in, d_out = w.d_in, w.d_out
        self.errors.require_dims(x.cols == d_in, "input width vs expert weights", (x.rows, x.cols), (d_in, d_out))
        if grouped_in:
            self.errors.require_dims(x.rows == num_slots, "grouped input rows vs slots", (x.rows,), (num_slots,))
        elif x.rows * fan_out != num_slots:
            raise ValueError(f"scattered input rows ({x.rows}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
        p = torch.from_numpy(np.ascontiguousarray(p_flat, dtype=x.dtype)).to(_DEVICE)
        with self._ref_errors():
            res = _k.scatter_combine(self._dev(x, "scatter_combine x"), self._dev(w, "scatter_combine w"),
                                     self._order(order), fan_out, p, combine_cols, grouped_in)
        self._credit(order, d_in, d_out)
        return self.core.Matrix(self._host(res))

    def group(self, x, order, weights=None, fan_out=1, out=None):
        if fan_out < 1:
            raise ValueError(f"fan_out must be >= 1, got {fan_out}")
        num_slots = order.num_slots
        if x.rows * fan_out != num_slots:
            raise ValueError(f"input rows ({x.rows}) * fan_out ({fan_out}) must equal T*k ({num_slots})")
        if weights is not None:
            self.errors.require_dims(weights.shape == (num_slots,), "slot weights", weights.shape, (num_slots,))
        if out is not None:
            self.errors.require_dims(out.rows == num_slots and out.cols == x.cols, "out buffer",
                                     (out.rows, out.cols), (num_slots, x.cols))
            if out.dtype != x.dtype:
                raise ValueError(f"out dtype {out.dtype} does not match input dtype {x.dtype}")
        wt = None
        if weights is not None:
            # the reference scales in the storage dtype (kernels.py:323-325)
            wt = torch.from_numpy(np.ascontiguousarray(weights, dtype=x.dtype)).to(_DEVICE)
        with self._ref_errors():
            res = _k.group(self._dev(x, "group x"), self._order(order), wt, fan_out)
        return self._into(out, res)

    def group_xty(self, xg, yg, order, tile=None):
        num_slots = order.num_slots
        self.errors.require_dims(xg.rows == num_slots, "grouped X rows vs slots", (xg.rows,), (num_slots,))
        self.errors.require_dims(yg.rows == num_slots, "grouped Y rows vs slots", (yg.rows,), (num_slots,))
        with self._ref_errors():
            dw = _k.group_xty(self._dev(xg, "group_xty xg"), self._dev(yg, "group_xty yg"), self._order(order))
        self._credit(order, xg.cols, yg.cols)
        return self.core.ExpertTensor(self._host(dw))

    def set_fault_injection(self, enabled: bool) -> None:
        _k.set_fault_injection(enabled)
        self.kernels._fault_inject = bool(enabled)

    def compute_grouped_order(self, routing, num_experts=None):
        e = routing.num_experts if num_experts is None else num_experts
        if e < routing.num_experts:
            raise ValueError(f"num_experts={e} smaller than routed id space {routing.num_experts}")
        flat = np.ascontiguousarray(routing.expert_idx.reshape(-1), dtype=np.int64)
        o, _, offsets, _ = _sort_ids(torch.from_numpy(flat).to(_DEVICE), e)
        return self.router.GroupedOrder(o=self._host(o).astype(np.int64),
                                        bin_offsets=self._host(offsets).astype(np.int64))

    def combine(self, p, y_hat):
        s, j = p.shape
        res = _k.combine(torch.from_numpy(np.ascontiguousarray(p, dtype=y_hat.dtype)).to(_DEVICE),
                         self._dev(y_hat, "combine y_hat").view(-1, y_hat.cols))
        return self.core.Matrix(self._host(res))

    def apply_activation(self, values, name):
        if name not in _k._lib.ACTIVATION_IDS:
            raise ValueError(f"unknown activation {name!r}; choose from {sorted(_k._lib.ACTIVATION_IDS)}")
        return self._host(_k.activation_kernel(self._dev(values, "apply_activation"), name, False))

    def activation_grad(self, pre, name):
        if name not in _k._lib.ACTIVATION_IDS:
            raise ValueError(f"unknown activation {name!r}; choose from {sorted(_k._lib.ACTIVATION_IDS)}")
        return self._host(_k.activation_kernel(self._dev(pre, "activation_grad"), name, True))


KERNEL_NAMES = ("scatter2scatter", "scatter_combine", "group", "group_xty", "set_fault_injection")


def install(ref) -> _Shim:
    """Rebind the hot-path names of an imported scattermlp package to the GPU kernels."""
    shim = _Shim(ref)
    for mod in (ref, shim.kernels, shim.pl):
        for name in KERNEL_NAMES:
            if hasattr(mod, name):
                setattr(mod, name, getattr(shim, name))
    ref.compute_grouped_order = shim.compute_grouped_order
    shim.pl._combine = shim.combine
    shim.layers.apply_activation = shim.apply_activation
    shim.layers.activation_grad = shim.activation_grad
    ref._gpu_shim = shim
    return shim
