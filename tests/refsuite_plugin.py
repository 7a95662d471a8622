"""pytest plugin: run the reference's own test files against the GPU kernels.

Loaded with ``-p refsuite_plugin`` by tests/test_reference_suite_gpu.py.  It
imports the vendored, unmodified ``scattermlp`` from baseline/_ref and calls
``paper_2403_08245_b200.refshim.install`` before any reference test module is
imported, so every ``from scattermlp import scatter2scatter`` (and the
reference's parallel_linear / moe_layers orchestration) resolves to the
C-ABI kernels.  SMOE_REFSUITE_FAULT=1 turns on the kernels' fault hook
(kernels.py:100-107 of the reference) before every test: the same suite must
then fail.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
for p in (str(REF), str(ROOT)):
    if p not in sys.path:
        sys.path.insert(0, p)

import scattermlp  # noqa: E402  (the vendored reference)

from paper_2403_08245_b200 import refshim  # noqa: E402

assert Path(scattermlp.__file__).resolve().is_relative_to(REF.resolve()), scattermlp.__file__
SHIM = refshim.install(scattermlp)
FAULT = os.environ.get("SMOE_REFSUITE_FAULT") == "1"


@pytest.fixture(autouse=True)
def _gpu_fault_hook():
    if FAULT:
        SHIM.set_fault_injection(True)
    yield
    if FAULT:
        SHIM.set_fault_injection(False)


def pytest_report_header(config):
    return [f"reference suite on the GPU kernels (scattermlp from {scattermlp.__file__}; fault={FAULT})"]
