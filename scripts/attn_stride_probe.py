"""Does the library SDPA take query / key / value / grad views in token-major
(b, S, heads, d) memory order without copies?  Times fwd+bwd at C3 for
head-contiguous inputs vs token-major strided views."""
import json
import torch
import torch.nn.functional as F

B, S, H, K, D = 8, 4096, 4, 4, 128
HQ = H * K


def run(strided):
    if strided:   # memory (b, S, heads, d); logical (b, heads, S, d)
        q = torch.randn(B, S, HQ, D, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_(True)
        k = torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_(True)
        v = torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_(True)
        do = torch.randn(B, S, HQ, D, device="cuda", dtype=torch.bfloat16).transpose(1, 2)
    else:
        q = torch.randn(B, HQ, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
        k = torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
        v = torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
        do = torch.randn(B, HQ, S, D, device="cuda", dtype=torch.bfloat16)

    def fb():
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        g = torch.autograd.grad(o, (q, k, v), do)
        return o, g

    for _ in range(3):
        o, g = fb()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fb()
    e1.record()
    torch.cuda.synchronize()
    return {"strided": strided, "ms": e0.elapsed_time(e1) / 10, "out_stride": list(o.stride()),
            "dq_stride": list(g[0].stride())}


print(json.dumps(run(False)))
print(json.dumps(run(True)))
