"""ctypes binding of libsmoe_b200.so (the C ABI declared in include/smoe_b200.h).

This is the FFI a maintainer of the reference would add: the reference is an
in-process NumPy package, so its "plugin boundary" is a Python call; the shim
here hands device pointers, sizes and the current CUDA stream to the C ABI.

There is deliberately no fallback: if the shared library is missing or fails
to load, every product entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# SMOE_LIB overrides the in-tree library (used by scripts/ab/ab.sh to A/B two builds
# of the same C ABI inside one GPU session).
LIB_PATH = Path(os.environ["SMOE_LIB"]) if os.environ.get("SMOE_LIB") else _PKG / "libsmoe_b200.so"

SMOE_OK, SMOE_EINVAL, SMOE_ESHAPE, SMOE_ECUDA, SMOE_ENOTSUP = range(5)
SMOE_F32, SMOE_BF16, SMOE_F64 = 0, 1, 2
ACTIVATION_IDS = {"gelu": 0, "relu": 1, "silu": 2}
ACT_IDENTITY = 3   # scatter2scatter_scaled only (routed linear with combine weights)
EPI_NONE, EPI_ACT, EPI_ACT_GRAD, EPI_ACT_ONLY, EPI_ACT_SCALED, EPI_ACT_GRAD_SCALED = 0, 1, 2, 3, 4, 5
ENGINE_IDS = {"auto": 0, "simt": 1, "tcgen05": 2}

_c = ctypes
_vp, _i64, _i32, _sz = _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_size_t

# name -> (restype, argtypes); the exact signatures of include/smoe_b200.h
SIGNATURES = {
    "smoe_get_last_error": (_c.c_char_p, []),
    "smoe_abi_version": (_c.c_int, []),
    "smoe_launch_count": (_c.c_uint64, []),
    "smoe_route_sort_workspace_bytes": (_sz, [_i64, _i32]),
    "smoe_route_sort": (_c.c_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "smoe_router_topk": (_c.c_int, [_vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "smoe_router_backward": (_c.c_int, [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "smoe_set_sm_reserve": (_c.c_int, [_i32]),
    "smoe_router_gate": (_c.c_int, [_vp, _i32, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "smoe_scatter2scatter": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _i32,
                                        _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "smoe_group_xty": (_c.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _i32, _vp, _i32, _vp]),
    "smoe_group": (_c.c_int, [_vp, _i64, _i64, _vp, _i64, _i32, _vp, _i32, _vp, _vp]),
    "smoe_combine": (_c.c_int, [_vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_combine_grad_p": (_c.c_int, [_vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_fanout_reduce": (_c.c_int, [_vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_fanout_reduce_grouped": (_c.c_int, [_vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_combine_grouped": (_c.c_int, [_vp, _vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_combine_grad_p_grouped": (_c.c_int, [_vp, _vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp]),
    "smoe_apply_activation": (_c.c_int, [_vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "smoe_ipc_handle_bytes": (_sz, []),
    "smoe_ipc_get_handle": (_c.c_int, [_vp, _vp, _c.POINTER(_c.c_int64)]),
    "smoe_ipc_open": (_c.c_int, [_vp, _c.POINTER(_c.c_void_p)]),
    "smoe_ipc_close": (_c.c_int, [_vp]),
    "smoe_ep_dispatch_rows": (_c.c_int, [_vp, _i64, _i64, _vp, _vp, _i32, _i32, _vp, _i64, _vp, _i32, _i32, _vp,
                                         _vp, _vp, _i32, _vp, _vp, _i64, _vp, _vp, _i32, _vp]),
    "smoe_ep_check_capacity": (_c.c_int, [_vp, _i32, _i64, _vp, _vp]),
    "smoe_ep_expert_gemm_gated": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp, _i32, _i32, _i32, _vp, _vp,
                                             _vp, _vp, _vp, _i32, _vp, _vp]),
    "smoe_ep_group_xty_gated": (_c.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp]),
    "smoe_ep_dp_return": (_c.c_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "smoe_ep_return_rows": (_c.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp]),
    "smoe_scatter2scatter_scaled": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _i32, _i32, _i32,
                                               _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "smoe_dp_parts": (_i32, [_i64]),
    "smoe_group_inv": (_c.c_int, [_vp, _i64, _i64, _vp, _i32, _vp, _i32, _vp, _vp]),
    "smoe_heads_to_grouped": (_c.c_int, [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _vp]),
    "smoe_scatter2scatter_heads": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _i32, _i32, _i32,
                                              _i32, _i32, _vp, _vp, _vp, _i32, _i64, _i32, _i32, _vp, _vp]),
    "smoe_grouped_to_heads": (_c.c_int, [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _vp]),
    "smoe_scale_grouped_rows": (_c.c_int, [_vp, _i64, _vp, _i64, _vp, _i32, _vp, _vp]),
    "smoe_dp_from_partials": (_c.c_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "smoe_ep_gemm_return": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp]),
    "smoe_ep_put": (_c.c_int, [_vp, _i64, _vp, _i64, _i32, _vp]),
    "smoe_ep_signal": (_c.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "smoe_ep_wait": (_c.c_int, [_vp, _i32, _i32, _vp, _i64, _vp, _vp]),
    "smoe_group_xty_scattered": (_c.c_int, [_vp, _i64, _i32, _i32, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _i64,
                                            _i64, _i64, _i32, _vp, _i32, _vp]),
    "smoe_scatter_combine": (_c.c_int, [_vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp, _i64, _i32,
                                        _vp, _i32, _i32, _i32, _vp, _vp, _i32, _vp]),
}

_lib = None
_load_error: str | None = None


class LibraryError(RuntimeError):
    """The native library is missing or a native call failed."""


ABI_VERSION = 4  # include/smoe_b200.h SMOE_ABI_VERSION


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raises if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        _load_error = f"{p} not found; run `python -m paper_2403_08245_b200.build` (no CPU fallback exists)"
        raise LibraryError(_load_error)
    lib = ctypes.CDLL(str(p))
    # SMOE_LIB_ALLOW_MISSING=1: A/B runs against an older build (SMOE_LIB) that
    # predates some entry points; those stay unbound and fail if called
    allow_missing = bool(os.environ.get("SMOE_LIB")) and os.environ.get("SMOE_LIB_ALLOW_MISSING") == "1"
    for name, (res, args) in SIGNATURES.items():
        if allow_missing and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.smoe_abi_version() != ABI_VERSION:
        raise LibraryError("libsmoe_b200.so ABI version mismatch")
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernels enqueued by libsmoe_b200.so since load (evidence for gpu_launches)."""
    return int(load().smoe_launch_count())


def last_error() -> str:
    return load().smoe_get_last_error().decode(errors="replace")


def check(status: int, what: str) -> None:
    """Map a C status onto the reference's exception classes (errors.py:3-19)."""
    if status == SMOE_OK:
        return
    from .errors import DimensionError

    msg = f"{what}: {last_error()}"
    if status == SMOE_ESHAPE:
        raise DimensionError(msg)
    if status == SMOE_EINVAL:
        raise ValueError(msg)
    if status == SMOE_ENOTSUP:
        raise NotImplementedError(msg)
    raise LibraryError(msg)
