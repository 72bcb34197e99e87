"""Minimal per-stage run for on-device debugging (not part of the product)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_06873_b200 import mec
dt = torch.bfloat16 if (len(sys.argv) < 2 or sys.argv[1] == "bf16") else torch.float32
I = torch.randn(1, 7, 7, 1, device="cuda").to(dt)
K = torch.randn(3, 3, 1, 16, device="cuda").to(dt)
L = mec.lower(I, 3, 3, 1, 1); torch.cuda.synchronize(); print("lower ok", flush=True)
O = mec.conv_forward(I, K, 1, 1, path=2); torch.cuda.synchronize(); print("conv ok", flush=True)
ref = torch.nn.functional.conv2d(I.float().permute(0,3,1,2), K.float().permute(3,2,0,1)).permute(0,2,3,1)
print("max err", (O.float()-ref).abs().max().item(), ref.abs().max().item())
