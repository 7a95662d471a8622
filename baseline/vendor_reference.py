"""Install the unmodified reference into baseline/_ref (git-ignored, shipped to the GPU box).

Runs only where /root/reference exists (the build container):

* ``scattermlp`` is installed with pip from a scratch copy of
  /root/reference/pkg (the reference tree is read-only) into baseline/_ref —
  the reference arm of bench.py and the CPU baseline time this package;
* the reference's own test files (/root/reference/pkg/tests) are copied to
  baseline/_ref/scattermlp_tests so tests/test_reference_suite_gpu.py can run
  them against the GPU kernels through paper_2403_08245_b200.refshim.

Nothing here is committed: baseline/_ref/ is in .gitignore.
"""
from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"


def vendor(force: bool = False) -> bool:
    """Returns True when baseline/_ref holds the package and the test files."""
    if not REF_SRC.exists():
        return (DEST / "scattermlp" / "__init__.py").exists()
    if force or not (DEST / "scattermlp" / "__init__.py").exists():
        with tempfile.TemporaryDirectory() as tmp:
            src = Path(tmp) / "pkg"
            shutil.copytree(REF_SRC, src)
            for p in src.rglob("*"):
                p.chmod(p.stat().st_mode | 0o200)
            subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                            "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(DEST), "--upgrade",
                            str(src)], check=True, capture_output=True)
    tests = DEST / "scattermlp_tests"
    if force or not tests.exists():
        if tests.exists():
            shutil.rmtree(tests)
        shutil.copytree(REF_SRC / "tests", tests)
        for p in tests.rglob("*"):
            p.chmod(p.stat().st_mode | 0o200)
        tests.chmod(tests.stat().st_mode | 0o200)
    return True


if __name__ == "__main__":
    print(vendor(force="--force" in sys.argv))
