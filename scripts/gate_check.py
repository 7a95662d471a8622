"""Gated vs ungated expert GEMMs on identical, already-resident inputs (bit identity)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08245_b200 as sm  # noqa: E402
from paper_2403_08245_b200 import _lib  # noqa: E402
from paper_2403_08245_b200 import kernels as K  # noqa: E402

lib = _lib.load()
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
for (n, cap, el, d, de) in [(1900, 2048, 4, 256, 512), (8000, 8192, 8, 1024, 512)]:
    h = (torch.rand(cap, de, device=dev, generator=g) - 0.5).bfloat16()
    dy = (torch.rand(cap, d, device=dev, generator=g) - 0.5).bfloat16()
    cuts = torch.sort(torch.randint(0, n, (el - 1,), generator=g, device=dev)).values
    off = torch.cat([torch.zeros(1, device=dev, dtype=torch.int64), cuts, torch.full((1,), n, device=dev, dtype=torch.int64)]).to(torch.int32)
    order = sm.GroupedOrder(o=torch.arange(cap, dtype=torch.int32, device=dev), bin_offsets=off, validate=False)
    ref = K.group_xty(h, dy, order)
    arrive = torch.full((el,), 1 << 40, dtype=torch.int64, device=dev)
    got = torch.empty_like(ref)
    st = lib.smoe_ep_group_xty_gated(h.data_ptr(), dy.data_ptr(), off.data_ptr(), el, cap, de, d, got.data_ptr(),
                                     arrive.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(st, "gated")
    torch.cuda.synchronize()
    print("xty", n, cap, "equal", torch.equal(ref, got), "maxdiff", (ref.float() - got.float()).abs().max().item())
    ref2 = K.group_xty(h[:n], dy[:n], sm.GroupedOrder(o=torch.arange(n, dtype=torch.int32, device=dev), bin_offsets=off, validate=False))
    print("xty n-vs-cap equal", torch.equal(ref, ref2))
