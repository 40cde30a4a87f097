import torch, time
x = torch.randn(123689472, device="cuda")
y = torch.empty_like(x)
def t(fn, n=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n*1e3
nb = x.numel()*4
for name, fn, bytes_ in [("max", lambda: x.max(), nb), ("sum", lambda: x.sum(), nb), ("copy", lambda: y.copy_(x), 2*nb), ("amax_abs", lambda: torch.linalg.vector_norm(x, float('inf')), nb)]:
    us = t(fn)
    print(f"{name}: {us:.1f} us  {bytes_/us/1e3:.0f} GB/s")
