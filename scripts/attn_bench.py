"""MoMHA attention core at C3 (B=8, seq 4096, 16 query heads = 4 KV heads x k=4, d_head=128, causal, bf16):
time of the library SDPA (enable_gqa) forward and forward+backward, CUDA events, after warm-up."""
import json
import torch
import torch.nn.functional as F

B, S, HKV, K, D = 8, 4096, 4, 4, 128
q = torch.randn(B, HKV * K, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
k = torch.randn(B, HKV, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
v = torch.randn(B, HKV, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
do = torch.randn(B, HKV * K, S, D, device="cuda", dtype=torch.bfloat16)
flop_fwd = 4.0 * B * HKV * K * S * S * D / 2


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


with torch.no_grad():
    ms_f = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True))


def fb():
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    torch.autograd.grad(o, (q, k, v), do)


ms_fb = timeit(fb)
print(json.dumps({"fwd_ms": ms_f, "fwd_tflops": flop_fwd / ms_f / 1e9, "fwd_bwd_ms": ms_fb,
                  "fwd_bwd_tflops": 3.5 * flop_fwd / ms_fb / 1e9}))
