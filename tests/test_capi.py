"""The C-ABI library loads and exports every symbol include/smoe_b200.h declares.

CPU-only: no compute call is made (there is no GPU in the build container).
"""
import re
from pathlib import Path

from conftest import ROOT

from paper_2403_08245_b200 import _lib

HEADER = ROOT / "include" / "smoe_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(smoe_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_loads():
    assert _lib.LIB_PATH.exists(), "run python -m paper_2403_08245_b200.build"
    lib = _lib.load()
    assert lib.smoe_abi_version() == _lib.ABI_VERSION == 4


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(names)


def test_argument_validation_without_a_gpu():
    """Validation runs before any device work, so bad calls fail cleanly on CPU."""
    lib = _lib.load()
    st = lib.smoe_scatter2scatter(None, 3, None, 2, 4, 4, None, None, 6, 0, 0, 0, 0, 1, 0, 0,
                                  None, None, None, 0, None)
    assert st == _lib.SMOE_EINVAL and "fan_out" in _lib.last_error()
    st = lib.smoe_scatter2scatter(None, 4, None, 2, 4, 4, None, None, 6, 2, 0, 0, 0, 1, 0, 0,
                                  None, None, None, 0, None)
    assert st == _lib.SMOE_EINVAL and "must equal T*k" in _lib.last_error()
    st = lib.smoe_scatter2scatter(None, 5, None, 2, 4, 4, None, None, 6, 1, 1, 0, 0, 1, 0, 0,
                                  None, None, None, 0, None)
    assert st == _lib.SMOE_ESHAPE
    st = lib.smoe_route_sort(None, 10, 0, None, None, None, None, None, 0, None)
    assert st == _lib.SMOE_EINVAL
    st = lib.smoe_group(None, 3, 4, None, 7, 2, None, 1, None, None)
    assert st == _lib.SMOE_EINVAL
    st = lib.smoe_combine(None, None, 4, 0, 8, 1, None, None)
    assert st == _lib.SMOE_EINVAL
    # zero-size work is a no-op success, no device touched
    assert lib.smoe_group(None, 0, 4, None, 0, 2, None, 1, None, None) == _lib.SMOE_OK
    # heads_to_grouped: slot count must equal batch * seq_len * k; null buffers rejected
    st = lib.smoe_heads_to_grouped(None, 2, 8, 4, 2, 64, None, 63, 1, None, None)
    assert st == _lib.SMOE_ESHAPE and "batch * seq_len * k" in _lib.last_error()
    st = lib.smoe_heads_to_grouped(None, 2, 8, 4, 2, 64, None, 64, 1, None, None)
    assert st == _lib.SMOE_EINVAL
    assert lib.smoe_heads_to_grouped(None, 0, 8, 4, 2, 64, None, 0, 1, None, None) == _lib.SMOE_OK
    # identity activation is accepted only by the scaled entry point
    st = lib.smoe_scatter2scatter(None, 6, None, 2, 4, 4, None, None, 6, 1, 1, 0, 0, 1, 0, 3,
                                  None, None, None, 0, None)
    assert st == _lib.SMOE_EINVAL and "activation" in _lib.last_error()


def test_status_maps_to_reference_exception_classes():
    import pytest

    from paper_2403_08245_b200.errors import DimensionError

    lib = _lib.load()
    lib.smoe_group(None, 3, 4, None, 7, 2, None, 1, None, None)
    with pytest.raises(ValueError):
        _lib.check(_lib.SMOE_EINVAL, "x")
    with pytest.raises(DimensionError):
        _lib.check(_lib.SMOE_ESHAPE, "x")


def test_sm100a_code_in_library():
    """The library carries sm_100a SASS (the only architecture built)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        import pytest
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bf16_never_falls_back_to_simt():
    """A bf16 GEMM the tcgen05 engine cannot take is refused (SMOE_ENOTSUP), never
    silently re-routed to the SIMT kernels.  Without a GPU the
    refusal is "no sm_100a device"; on the B200 it names the unsupported shape
    (tests/test_kernels_gpu.py::test_bf16_unsupported_shape_is_refused)."""
    lib = _lib.load()
    # d_out = 12 (not a multiple of 8), scattered in/out, bf16, engine AUTO; buffers are fake
    fake = 1 << 20
    st = lib.smoe_scatter2scatter(fake, 4, fake, 2, 16, 12, fake, fake, 8, 2, 0, 0, 0, _lib.SMOE_BF16, 0, 0,
                                  fake, None, None, _lib.ENGINE_IDS["auto"], None)
    assert st == _lib.SMOE_ENOTSUP, _lib.last_error()
    st = lib.smoe_group_xty(fake, fake, fake, 2, 8, 16, 12, _lib.SMOE_BF16, fake, _lib.ENGINE_IDS["auto"], None)
    assert st == _lib.SMOE_ENOTSUP, _lib.last_error()
