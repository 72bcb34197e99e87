import torch
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").normal_()
def t(fn, it=10):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
ms = t(lambda: x.sum(dtype=torch.float32))
print(f"torch sum (pure read) of 2 GiB: {2*2**30/ms/1e6:.0f} GB/s")
y = torch.empty_like(x)
ms = t(lambda: y.copy_(x))
print(f"torch copy 2 GiB: {2*2*2**30/ms/1e6:.0f} GB/s")
ms = t(lambda: y.fill_(1.0))
print(f"torch fill (pure write) 2 GiB: {2*2**30/ms/1e6:.0f} GB/s")
