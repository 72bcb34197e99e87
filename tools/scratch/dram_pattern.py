"""DRAM read efficiency of 128-byte row pieces at a large stride (the TMA box
pattern of the window GEMMs over a pitched L) vs contiguous, with torch copies."""
import torch
dev = "cuda"
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
pitch = 43008  # C2 L row (elements)
rows = 14208 * 2
A = torch.randn(rows, pitch, device=dev).to(torch.bfloat16)  # 2.4 GB
for w in (64, 128, 256, 512):
    sub = A[:, :w]
    out = torch.empty(rows, w, device=dev, dtype=torch.bfloat16)
    ms = t(lambda: out.copy_(sub))
    byts = 2 * rows * w * 2
    print(f"strided rows of {w*2} B at {pitch*2} B stride: {byts/ms/1e6:.0f} GB/s (read+write)")
flat = A.view(-1)[: rows * 64]
out = torch.empty_like(flat)
ms = t(lambda: out.copy_(flat))
print(f"contiguous same bytes: {2*flat.numel()*2/ms/1e6:.0f} GB/s")
big = A.view(-1)
out2 = torch.empty_like(big)
ms = t(lambda: out2.copy_(big))
print(f"contiguous 2.4 GB: {2*big.numel()*2/ms/1e6:.0f} GB/s")
