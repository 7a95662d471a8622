import torch, time
b, S, k, h, d = 8, 4096, 4, 4, 128
q = torch.randn(b * S * k, h * d, device="cuda").bfloat16()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
f1 = lambda: q.view(b, S, k, h, d).permute(0, 3, 2, 1, 4).reshape(b, h * k, S, d)
def f2():
    c = q.view(torch.complex128).view(b, S, k, h, d // 8).permute(0, 3, 2, 1, 4).reshape(b, h * k, S, d // 8)
    return c.view(torch.bfloat16)
def f3():
    c = q.view(torch.int64).view(b, S, k, h, d // 4).permute(0, 3, 2, 1, 4).reshape(b, h * k, S, d // 4)
    return c.view(torch.bfloat16)
print("bf16 permute copy ms", t(f1)); print("complex128 ms", t(f2)); print("int64 ms", t(f3))
assert torch.equal(f1(), f2()) and torch.equal(f1(), f3())
print("equal ok", f2().shape, f2().is_contiguous())
