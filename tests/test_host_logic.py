"""Host-side logic of the shim that runs without a GPU: validation, routing
construction, error classes — mirroring the reference's own argument checks
(router.py:38-60, kernels.py:46-58/:172-197, parallel_linear.py:76-82)."""
import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm
from paper_2403_08245_b200.errors import DimensionError


def test_tile_config_validation():
    sm.TileConfig(4, 8, 8, 2)
    with pytest.raises(ValueError):
        sm.TileConfig(tile_rows=0)


def test_layout_constants():
    assert sm.SCATTERED_TO_GROUPED == sm.LayoutFlag(False, True)
    assert sm.GROUPED_TO_SCATTERED == sm.LayoutFlag(True, False)


def test_softmax_and_topk_known_values():
    """test_router.py:22-47 vectors, computed by the torch gate glue on CPU."""
    g = sm.softmax_rows(torch.tensor([[2.0, 1.0, 0.0, -1.0]]))
    np.testing.assert_allclose(g[0].numpy(), [0.64391426, 0.23688282, 0.08714432, 0.0320586], atol=1e-6)
    r = sm.topk_select(g, 2)
    assert r.expert_idx[0].tolist() == [0, 1]
    np.testing.assert_allclose(r.p[0].numpy(), [0.73105858, 0.26894142], atol=1e-6)
    ties = sm.topk_select(sm.softmax_rows(torch.zeros(3, 5)), 2)
    assert ties.expert_idx.tolist() == [[0, 1]] * 3


def test_routing_validation_errors():
    with pytest.raises(ValueError, match="duplicate"):
        sm.assignment_routing(np.array([[1, 1]]), 3)
    with pytest.raises(ValueError, match="expert ids"):
        sm.assignment_routing(np.array([[0, 3]]), 3)
    with pytest.raises(ValueError, match="k must be"):
        sm.RoutingResult(torch.zeros(2, 4, dtype=torch.int64), torch.zeros(2, 4), torch.zeros(2, 3))
    with pytest.raises(DimensionError):
        sm.RoutingResult(torch.zeros(2, 2, dtype=torch.int64), torch.zeros(3, 2), torch.zeros(2, 3))
    r = sm.assignment_routing(np.array([[0, 2], [1, 0]]), 3, p=np.array([[3.0, 1.0], [1.0, 1.0]]))
    np.testing.assert_allclose(r.p.numpy(), [[0.75, 0.25], [0.5, 0.5]])


def test_grouped_order_validation():
    with pytest.raises(ValueError):
        sm.GroupedOrder(o=torch.arange(4), bin_offsets=torch.tensor([0, 2, 3]))
    with pytest.raises(ValueError):
        sm.GroupedOrder(o=torch.arange(4), bin_offsets=torch.tensor([0, 3, 2, 4]))
    g = sm.GroupedOrder(o=torch.tensor([0, 3, 2, 1]), bin_offsets=torch.tensor([0, 2, 3, 4]))
    assert g.bin_counts.tolist() == [2, 1, 1]
    assert g.inverse().tolist() == [0, 3, 2, 1]
    assert g.expert_offsets.tolist() == [2, 3, 4]


def _order(idx, e):
    from oracle.scattermlp_oracle import compute_grouped_order
    o, off = compute_grouped_order(np.asarray(idx), e)
    return sm.GroupedOrder(o=torch.from_numpy(o).int(), bin_offsets=torch.from_numpy(off).int())


def test_kernel_shape_errors_match_reference():
    """kernels.py:172-197 error classes, raised before any device work."""
    order = _order([[0, 1], [1, 0], [2, 1]], 3)
    w = torch.zeros(3, 4, 5)
    with pytest.raises(ValueError, match="fan_out"):
        sm.scatter2scatter(torch.zeros(3, 4), w, order, 0)
    with pytest.raises(ValueError, match="must equal T"):
        sm.scatter2scatter(torch.zeros(4, 4), w, order, 2)
    with pytest.raises(DimensionError):
        sm.scatter2scatter(torch.zeros(3, 7), w, order, 2)
    with pytest.raises(DimensionError):
        sm.scatter2scatter(torch.zeros(5, 4), w, order, 1, sm.GROUPED_TO_GROUPED)
    with pytest.raises(DimensionError):
        sm.scatter2scatter(torch.zeros(3, 4), torch.zeros(2, 4, 5), order, 2)
    with pytest.raises(DimensionError):
        sm.scatter2scatter(torch.zeros(3, 4), w, order, 2, out=torch.zeros(6, 4))
    with pytest.raises(ValueError, match="dtype"):
        sm.scatter2scatter(torch.zeros(3, 4), w, order, 2, out=torch.zeros(6, 5, dtype=torch.float64))
    with pytest.raises(ValueError, match="CUDA"):
        sm.scatter2scatter(torch.zeros(3, 4), w, order, 2)
    with pytest.raises(DimensionError):
        sm.group_xty(torch.zeros(5, 2), torch.zeros(6, 2), order)
    with pytest.raises(ValueError, match="fan_out"):
        sm.group(torch.zeros(3, 4), order, fan_out=0)


def test_parallel_linear_argument_errors():
    order = _order([[0, 1], [1, 0], [2, 1]], 3)
    w = torch.zeros(3, 4, 5)
    with pytest.raises(ValueError, match="2-D"):
        sm.parallel_linear_forward(torch.zeros(3, 4), w, order, p=torch.zeros(6), fan_out=2)
    with pytest.raises(ValueError, match="cover"):
        sm.parallel_linear_forward(torch.zeros(3, 4), w, order, p=torch.zeros(2, 2), fan_out=2)
    with pytest.raises(ValueError, match="grouped_out"):
        sm.parallel_linear_forward(torch.zeros(3, 4), w, order, p=torch.zeros(3, 2), fan_out=2,
                                   layout=sm.SCATTERED_TO_GROUPED)


def test_config_validation():
    with pytest.raises(ValueError):
        sm.SmoeMlpConfig(d_model=4, d_expert=4, num_experts=2, k=3)
    with pytest.raises(ValueError):
        sm.SmoeMlpConfig(d_model=4, d_expert=4, num_experts=2, k=1, activation="tanh")
    with pytest.raises(ValueError):
        sm.MomhaConfig(d_model=8, d_head=2, num_heads=3, heads_per_expert=2, num_experts=2, k=2)
    assert sm.MomhaConfig(d_model=8, d_head=2, num_heads=4, heads_per_expert=2, num_experts=2, k=2).d_proj == 4


def test_mac_counter_is_padding_free_arithmetic():
    sm.reset_mac_count()
    sm.add_macs(7)
    assert sm.mac_count() == 7
    sm.reset_mac_count()


def test_bench_reference_arm_json_line():
    """bench.py --impl reference (the unmodified reference from baseline/_ref on the
    host CPU; the oracle port only when baseline/_ref is absent) prints the
    contract's JSON line: metric/unit/higher_is_better, impl, cpu_baseline and
    an e2e object with zero transfer bytes; under torchrun only rank 0 prints."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--config", "C0",
                          "--steps", "1", "--warmup", "0", "--ref-tokens", "16"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["higher_is_better"] is True
    from baseline import cpu_reference
    want_kind = "reference" if cpu_reference.available() else "port"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == want_kind and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    env = dict(__import__("os").environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out1 = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--config", "C0",
                           "--steps", "1", "--warmup", "0", "--ref-tokens", "16"],
                          capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out1.returncode == 0 and not [ln for ln in out1.stdout.splitlines() if ln.startswith("{")]
