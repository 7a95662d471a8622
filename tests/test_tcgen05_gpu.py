"""tcgen05 engines (CTA-pair default and single-CTA) vs the SIMT engine.

Both engines compute the same fp32-accumulated products from bf16 inputs, so
they agree to bf16 rounding (one ulp on a few elements).  Shapes probe the
masking and scheduling edges: bins smaller than one tile, empty experts,
all tokens on one expert, K not a multiple of 64, N not a multiple of 256,
fan-out 1..4, E up to 64.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2403_08245_b200 as sm

pytestmark = pytest.mark.gpu

CASES = [
    # T, k, E, d_in, d_out, flavor
    (1, 1, 1, 64, 256, "gate"),
    (7, 2, 4, 72, 136, "gate"),
    (300, 3, 5, 264, 520, "skip"),
    (513, 2, 8, 128, 256, "one"),
    (2000, 4, 64, 256, 128, "gate"),
    (4096, 2, 8, 1032, 1800, "gate"),
]


def _routing(t, k, e, flavor, g):
    if flavor == "one":
        ids = torch.arange(k, device="cuda").repeat(t, 1)
    else:
        e_eff = e - 1 if (flavor == "skip" and e > k) else e
        ids = torch.stack([torch.randperm(e_eff, generator=g)[:k] for _ in range(t)]).cuda()
    p = torch.rand(t, k, device="cuda") + 0.1
    return sm.RoutingResult(ids, p, torch.zeros(t, e, device="cuda"), renormalized=False, validate=False)


def _rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("case", CASES)
def test_engines_agree(case):
    t, k, e, d_in, d_out, flavor = case
    g = torch.Generator().manual_seed(hash(case) % 2**31)
    routing = _routing(t, k, e, flavor, g)
    order = sm.compute_grouped_order(routing)
    n = t * k
    xs = (torch.rand(t, d_in, device="cuda") * 2 - 1).bfloat16()
    xg = (torch.rand(n, d_in, device="cuda") * 2 - 1).bfloat16()
    w = ((torch.rand(e, d_in, d_out, device="cuda") * 2 - 1) / d_in ** 0.5).bfloat16()
    wt = ((torch.rand(e, d_out, d_in, device="cuda") * 2 - 1) / d_in ** 0.5).bfloat16()
    for x, lay, fan in ((xs, sm.SCATTERED_TO_GROUPED, k), (xs, sm.SCATTERED_TO_SCATTERED, k),
                        (xg, sm.GROUPED_TO_SCATTERED, 1), (xg, sm.GROUPED_TO_GROUPED, 1)):
        for tr, ww in ((False, w), (True, wt)):
            a = sm.scatter2scatter(x, ww, order, fan, lay, transpose_w=tr, engine="simt")
            b = sm.scatter2scatter(x, ww, order, fan, lay, transpose_w=tr, engine="tcgen05")
            assert _rel(b, a) < 1e-3, (case, lay, tr)
    yg = (torch.rand(n, d_out, device="cuda") * 2 - 1).bfloat16()
    a = sm.group_xty(xg, yg, order, engine="simt")
    b = sm.group_xty(xg, yg, order, engine="tcgen05")
    assert _rel(b, a) < 1e-3, case
    counts = order.bin_counts.cpu()
    for ee in torch.nonzero(counts == 0).flatten().tolist():
        assert float(b[ee].float().abs().max()) == 0.0


def test_single_cta_engine_matches_pair_engine():
    """SMOE_TC_CTAS=1 (single-CTA kernels) vs the default CTA-pair kernels, in a subprocess."""
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2403_08245_b200 as sm
torch.manual_seed(0)
t, k, e, d, de = 1500, 2, 8, 256, 512
ids = torch.stack([torch.randperm(e)[:k] for _ in range(t)]).cuda()
r = sm.RoutingResult(ids, torch.rand(t, k, device='cuda'), torch.zeros(t, e, device='cuda'), renormalized=False, validate=False)
o = sm.compute_grouped_order(r)
x = (torch.rand(t, d, device='cuda') * 2 - 1).bfloat16()
w = ((torch.rand(e, d, de, device='cuda') * 2 - 1) / 16).bfloat16()
y = sm.scatter2scatter(x, w, o, k, sm.SCATTERED_TO_GROUPED, engine='tcgen05')
dw = sm.group_xty(y, y, o, engine='tcgen05')
torch.save((y.cpu(), dw.cpu()), sys.argv[1])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for ctas in ("2", "1"):
        path = f"/tmp/smoe_tc_{ctas}.pt"
        env = dict(os.environ, SMOE_TC_CTAS=ctas, SMOE_TC_SERP="0")   # same K order in both engines
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs.append(torch.load(path))
    (y2, dw2), (y1, dw1) = outs
    assert torch.equal(y1, y2)          # same products, same fp32 accumulation order per K block
    assert _rel(dw1, dw2) < 1e-3


def test_tma_store_epilogue_matches_direct():
    """SMOE_TC_EPI=all (staged TMA-store epilogue on every grouped-output kernel)
    is bit-identical to the default direct-store epilogue: bin tails, column
    tails, fused activation / activation-grad outputs and group_xty."""
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2403_08245_b200 as sm
torch.manual_seed(1)
t, k, e, d, de = 1900, 2, 8, 264, 584
ids = torch.stack([torch.randperm(e)[:k] for _ in range(t)]).cuda()
r = sm.RoutingResult(ids, torch.rand(t, k, device='cuda'), torch.zeros(t, e, device='cuda'), renormalized=False, validate=False)
o = sm.compute_grouped_order(r)
x = (torch.rand(t * k, d, device='cuda') * 2 - 1).bfloat16()
w = ((torch.rand(e, d, de, device='cuda') * 2 - 1) / 16).bfloat16()
h = torch.empty(t * k, de, device='cuda', dtype=torch.bfloat16)
a = torch.empty_like(h)
sm.scatter2scatter(x, w, o, 1, sm.GROUPED_TO_GROUPED, out=h, activation='gelu', act_out=a, engine='tcgen05')
g = sm.scatter2scatter(x, w, o, 1, sm.GROUPED_TO_GROUPED, activation='gelu', act_grad_of=h, engine='tcgen05')
dw = sm.group_xty(x, h, o, engine='tcgen05')
torch.save((h.cpu(), a.cpu(), g.cpu(), dw.cpu()), sys.argv[1])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("default", "all"):
        path = f"/tmp/smoe_epi_{mode}.pt"
        env = dict(os.environ, SMOE_TC_EPI=mode)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs.append(torch.load(path))
    for u, v in zip(*outs):
        assert torch.equal(u, v)


def test_wide_tiles_match_256_row_tiles(tmp_path):
    """Wide 512 x 256 pair tiles (SMOE_TC_WIDE=1: two M=256 MMAs per B stage,
    grouped MMA issue) are bit-identical to the 256 x 256 tiles (SMOE_TC_WIDE=0):
    the same K16 products accumulate in the same order per output element.
    Covers bins shorter than half a wide tile (second MMA skipped), bins that
    are not multiples of 512, empty experts, K tails of the grouped-K kernel,
    N tails, the scaled / activation / act-grad epilogues, scattered outputs,
    and both group-issue depths (SMOE_TC_WIDE_DEFER=1 and 4)."""
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2403_08245_b200 as sm
torch.manual_seed(2)
outs = []
for (t, k, e, d, de) in ((2100, 2, 8, 264, 584), (700, 3, 16, 136, 1032), (37, 1, 4, 64, 256)):
    ids = torch.stack([torch.randperm(e - 1)[:k] for _ in range(t)]).cuda()   # expert e-1 stays empty
    p = torch.rand(t, k, device='cuda') + 0.1
    r = sm.RoutingResult(ids, p, torch.zeros(t, e, device='cuda'), renormalized=False, validate=False)
    o = sm.compute_grouped_order(r)
    n = t * k
    xg = (torch.rand(n, d, device='cuda') * 2 - 1).bfloat16()
    w = ((torch.rand(e, d, de, device='cuda') * 2 - 1) / 16).bfloat16()
    wt = ((torch.rand(e, de, d, device='cuda') * 2 - 1) / 16).bfloat16()
    h = torch.empty(n, de, device='cuda', dtype=torch.bfloat16)
    a = torch.empty_like(h)
    sm.scatter2scatter(xg, w, o, 1, sm.GROUPED_TO_GROUPED, out=h, activation='gelu', act_out=a, engine='tcgen05')
    outs += [h, a]
    outs.append(sm.scatter2scatter(xg, w, o, 1, sm.GROUPED_TO_SCATTERED, engine='tcgen05'))
    outs.append(sm.scatter2scatter(h, wt, o, 1, sm.GROUPED_TO_SCATTERED, engine='tcgen05'))
    outs.append(sm.scatter2scatter(xg, wt, o, 1, sm.GROUPED_TO_GROUPED, transpose_w=True, engine='tcgen05'))
    outs.append(sm.scatter2scatter(xg, w, o, 1, sm.GROUPED_TO_GROUPED, activation='gelu', act_grad_of=h,
                                   engine='tcgen05'))
    pf = p.reshape(-1).float().contiguous()
    outs.append(sm.kernels.scatter2scatter_scaled(xg, w, o, 1, sm.GROUPED_TO_GROUPED, row_scale=pf,
                                                  activation='gelu', out=torch.empty_like(h), act_out=a.clone()))
    outs.append(sm.group_xty(xg, h, o, engine='tcgen05'))
    outs.append(sm.group_xty(h, xg, o, engine='tcgen05'))
    outs.append(sm.scatter_combine(h, wt, o, 1, p.reshape(-1).contiguous(), k, True, engine='tcgen05'))
    if k <= 2:   # fused combine epilogue: two fp32 additions into a zeroed row commute
        sm.kernels._COMBINE_FUSED = '1'
        outs.append(sm.scatter_combine(h, wt, o, 1, p.reshape(-1).contiguous(), k, True, engine='tcgen05'))
        sm.kernels._COMBINE_FUSED = 'auto'
torch.save([x.cpu() for x in outs], sys.argv[1])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for tag, env_add in (("off", {"SMOE_TC_WIDE": "0"}), ("wide4", {"SMOE_TC_WIDE": "1"}),
                         ("wide1", {"SMOE_TC_WIDE": "1", "SMOE_TC_WIDE_DEFER": "1"}),
                         # the wave-lockstep gate only reorders issue in time
                         ("lockstep", {"SMOE_TC_WIDE": "1", "SMOE_TC_SYNC": "2", "SMOE_TC_SYNC_SLACK": "1"})):
        path = str(tmp_path / f"wide_{tag}.pt")
        # serpentine K order off: it reverses tiles by their index, which the tile shape changes
        subprocess.run([sys.executable, "-c", code, path], check=True,
                       env=dict(os.environ, SMOE_TC_SERP="0", **env_add), timeout=300)
        runs[tag] = torch.load(path)
    for tag in ("wide4", "wide1", "lockstep"):
        for i, (u, v) in enumerate(zip(runs["off"], runs[tag])):
            assert torch.equal(u, v), (tag, i)


def test_serpentine_k_order(tmp_path):
    """SMOE_TC_SERP: tiles of odd 74-tile waves (counted within their expert)
    stream K last-to-first.  Only the fp32 accumulation order changes: the
    results match the forward order to rounding, differ somewhere (the reversal
    ran), and are deterministic run to run."""
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2403_08245_b200 as sm
torch.manual_seed(4)
t, k, e, d, de = 8192, 2, 2, 328, 4872       # ~8192 rows per expert: > 74 tiles per expert
ids = torch.stack([torch.randperm(e)[:k] for _ in range(t)]).cuda()
r = sm.RoutingResult(ids, torch.rand(t, k, device='cuda'), torch.zeros(t, e, device='cuda'), renormalized=False, validate=False)
o = sm.compute_grouped_order(r)
n = t * k
xg = (torch.rand(n, d, device='cuda') * 2 - 1).bfloat16()
w = ((torch.rand(e, d, de, device='cuda') * 2 - 1) / 16).bfloat16()
h = torch.empty(n, de, device='cuda', dtype=torch.bfloat16)
a = torch.empty_like(h)
sm.scatter2scatter(xg, w, o, 1, sm.GROUPED_TO_GROUPED, out=h, activation='gelu', act_out=a, engine='tcgen05')
outs = [h, a, sm.scatter2scatter(h, w, o, 1, sm.GROUPED_TO_SCATTERED, transpose_w=True, engine='tcgen05'),
        sm.group_xty(xg, h, o, engine='tcgen05'), sm.group_xty(h, xg, o, engine='tcgen05')]
torch.save([x.cpu() for x in outs], sys.argv[1])
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for tag, serp in (("fwd", "0"), ("serp", "2"), ("serp_again", "2")):
        path = str(tmp_path / f"serp_{tag}.pt")
        subprocess.run([sys.executable, "-c", code, path], check=True, env=dict(os.environ, SMOE_TC_SERP=serp),
                       timeout=300)
        runs[tag] = torch.load(path)
    differs = False
    for i, (u, v, w_) in enumerate(zip(runs["fwd"], runs["serp"], runs["serp_again"])):
        assert torch.equal(v, w_), i
        assert _rel(v, u) < 2e-3, (i, _rel(v, u))
        differs = differs or not torch.equal(u, v)
    assert differs
