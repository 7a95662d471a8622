"""Zero-padding memory on the GPU.

The reference asserts padding-freedom on its logical ledger: the backward with
seeded scratch allocates no T*k-row buffer (test_parallel_linear.py:175-200,
test_moe_layers.py:190-201) and the fused pipeline never holds a padded bin
(test_oracle_accounting.py:148-158).  The GPU analogue uses the caching
allocator's statistics (every byte the library path allocates goes through
torch; the C-ABI itself never allocates):

* forward (training) allocates exactly its analytic outputs — the grouped
  pre-activation and activation (n x d_expert each), the slot-ordered layer-2
  output kept for the backward (n x d_model) and Y — and no buffer of the padded
  size sum_e ceil(count_e / 128) * 128 rows;
* backward allocates only its outputs (dX, dW1, dW2, dp) plus the dp partials
  (n x parts fp32, < 6 % of one slot buffer) — no new n-row activation buffer;
* the fused step's peak stays well under the padded group-copy baseline the
  paper compares against (66.2 % of Megablocks in training),
  at C1 and at the paper's own configuration (E=32, k=4, T=30*2048,
  d_model=4096, d_expert=2048).
"""
import sys
from pathlib import Path

import pytest
import torch

import paper_2403_08245_b200 as sm

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))

CONFIGS = {"C1": (32768, 4096, 14336, 8, 2), "paper_E32_k4": (61440, 4096, 2048, 32, 4)}
MB = 1 << 20


def _problem(t, d, de, e, k, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    dy = (torch.rand(t, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    w1 = ((torch.rand(e, d, de, device="cuda", generator=g) * 2 - 1) / d ** 0.5).bfloat16()
    w2 = ((torch.rand(e, de, d, device="cuda", generator=g) * 2 - 1) / de ** 0.5).bfloat16()
    routing = sm.topk_select(torch.softmax(torch.randn(t, e, device="cuda", generator=g), 1), k)
    order = sm.compute_grouped_order(routing)
    return x, dy, w1, w2, routing, order


def _peak_delta(fn):
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    out = fn()
    torch.cuda.synchronize()
    return torch.cuda.max_memory_allocated() - base, torch.cuda.memory_allocated() - base, out


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
@pytest.mark.parametrize("scaled", [True, False])
def test_fused_step_allocates_only_its_outputs(cfg, scaled):
    t, d, de, e, k = CONFIGS[cfg]
    n = t * k
    x, dy, w1, w2, routing, order = _problem(t, d, de, e, k)
    prev = sm.moe_layers.set_scaled(scaled)
    try:
        fwd_peak, fwd_live, (y, ctx) = _peak_delta(lambda: sm.smoe_mlp_forward(x, w1, w2, routing, order))
        bwd_peak, _, g = _peak_delta(lambda: sm.smoe_mlp_backward(ctx, dy))
    finally:
        sm.moe_layers.set_scaled(prev)
    bf = 2
    # forward outputs: h_pre, act (n x de each), the slot-ordered layer-2 output (n x d), Y, p per slot
    fwd_budget = 2 * n * de * bf + n * d * bf + t * d * bf + n * 4
    assert fwd_live <= fwd_budget + 4 * MB, (fwd_live, fwd_budget)
    assert fwd_peak <= fwd_budget + 4 * MB, (fwd_peak, fwd_budget)
    # backward: dX, dW1, dW2, dp (+ dp partials and p per slot); every slot buffer is reused
    parts = n * sm.kernels.dp_parts(de) * 4 if scaled else 0
    bwd_budget = t * d * bf + 2 * e * d * de * bf + t * k * 4 + parts + n * 4
    assert bwd_peak <= bwd_budget + 4 * MB, (bwd_peak, bwd_budget)
    assert parts < 0.06 * n * d * bf
    assert g.dx.shape == (t, d) and y.shape == (t, d)


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
def test_fused_peak_below_padded_baseline(cfg):
    """PAPER.md:358-363 (66.2 % of the padded baseline in training) reproduced in direction."""
    from memory_footprint import fused_step, measure, padded_step

    t, d, de, e, k = CONFIGS[cfg]
    x, dy, w1, w2, routing, order = _problem(t, d, de, e, k)
    fused, _ = measure(fused_step, x, w1, w2, routing, order, dy)
    padded, (pad_rows, _) = measure(padded_step, x, w1, w2, routing, order, dy)
    assert pad_rows > 0
    assert fused < 0.8 * padded, (fused / 1e9, padded / 1e9)
