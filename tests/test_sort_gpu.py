"""K1 parity: the GPU stable counting sort is bit-exact against the reference.

Pinned on the reference's own KATs (test_router.py:58-77), on
reference-generated property cases (tests/golden/routing.npz) and at every
BASELINE.json size through the oracle's stable argsort.
"""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import scattermlp_oracle as orc

pytestmark = pytest.mark.gpu


def _check(idx, e):
    from gpu_util import order_of
    idx = np.asarray(idx, dtype=np.int64)
    g = order_of(idx, e)
    o, off = orc.compute_grouped_order(idx, e)
    assert np.array_equal(g.o.cpu().numpy().astype(np.int64), o)
    assert np.array_equal(g.bin_offsets.cpu().numpy().astype(np.int64), off)
    flat = idx.reshape(-1)
    assert np.array_equal(g.sorted_expert_idxs.cpu().numpy(), flat[o])
    assert np.array_equal(g.inverse().cpu().numpy().astype(np.int64), orc.inverse(o))
    return g


def test_reference_known_answers():
    gold = load_golden("routing")
    for i in range(int(gold["num_kats"])):
        g = _check(gold[f"kat{i}_idx"], int(gold[f"kat{i}_E"]))
        assert np.array_equal(g.o.cpu().numpy(), gold[f"kat{i}_o"])
        assert np.array_equal(g.bin_offsets.cpu().numpy(), gold[f"kat{i}_off"])


def test_reference_property_cases():
    gold = load_golden("routing")
    for j in range(int(gold["num_cases"])):
        g = _check(gold[f"case{j}_idx"], int(gold[f"case{j}_E"]))
        assert np.array_equal(g.o.cpu().numpy(), gold[f"case{j}_o"])


@pytest.mark.parametrize("t,k,e", [(4096, 2, 8), (32768, 2, 8), (32768, 8, 64), (32768, 4, 16),
                                   (5000, 3, 7), (1, 1, 1), (4097, 1, 1), (70000, 2, 1024),
                                   (300001, 4, 1024), (600000, 2, 5), (262145, 4, 2),
                                   (70001, 3, 256), (50001, 1, 255), (1 << 20, 2, 8), (12289, 1, 3)])
def test_baseline_sizes_random(t, k, e):
    rng = np.random.default_rng(t + k + e)
    idx = np.stack([rng.permutation(e)[:k] for _ in range(min(t, 2000))])
    idx = np.resize(idx, (t, k))
    _check(idx, e)


def test_skewed_and_empty_bins():
    t, k, e = 40000, 2, 16
    _check(np.tile(np.arange(k), (t, 1)), e)                        # all_to_one
    rng = np.random.default_rng(0)
    zipf = np.minimum(rng.zipf(1.3, size=t * k) - 1, e - 1).reshape(t, k)
    _check(zipf, e)                                                # skewed (dups allowed in sort)
    _check(np.zeros((0, 2), dtype=np.int64), 4)                    # empty routing


def test_large_n_sixteen_million():
    n, e = 1 << 24, 64
    rng = np.random.default_rng(1)
    idx = rng.integers(0, e, size=(n // 8, 8))
    _check(idx, e)


def test_flatten_and_sort_api():
    import paper_2403_08245_b200 as sm
    ids = torch.tensor([[0, 2], [1, 0]], device="cuda")
    se, ss, offs = sm.flatten_and_sort(ids, 3, return_offsets=True)
    assert ss.tolist() == [0, 3, 2, 1]
    assert se.tolist() == [0, 0, 1, 2]
    assert offs.tolist() == [2, 3, 4]


def test_two_pass_path_same_suite():
    """The same cases through the two-pass kernels (SMOE_SORT_ONEPASS=0): the
    one-pass cooperative kernel is the default whenever a chunk fits in shared
    memory, the two-pass path serves larger n and E > 256."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    if os.environ.get("SMOE_SORT_ONEPASS") == "0":
        pytest.skip("already the two-pass run")
    here = Path(__file__).resolve()
    env = dict(os.environ, SMOE_SORT_ONEPASS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", str(here), "-m", "gpu",
                        "-k", "not two_pass"], cwd=here.parent.parent, env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
