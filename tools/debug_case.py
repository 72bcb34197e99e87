"""Run one conv shape through the C ABI (debugging aid). args: i_n i_h i_w i_c k_h k_w k_c s_h s_w [path] [dtype]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_06873_b200 import mec
a = [int(x) for x in sys.argv[1:10]]
path = int(sys.argv[10]) if len(sys.argv) > 10 else 0
dt = torch.float32 if (len(sys.argv) > 11 and sys.argv[11] == "tf32") else torch.bfloat16
i_n, i_h, i_w, i_c, k_h, k_w, k_c, s_h, s_w = a
I = torch.randn(i_n, i_h, i_w, i_c, device="cuda").to(dt)
K = torch.randn(k_h, k_w, i_c, k_c, device="cuda").to(dt)
O, p = mec.conv_forward(I, K, s_h, s_w, path=path, return_path=True)
torch.cuda.synchronize()
ref = torch.nn.functional.conv2d(I.double().permute(0,3,1,2), K.double().permute(3,2,0,1), stride=(s_h, s_w)).permute(0,2,3,1)
print("path", p, "max err", (O.double()-ref).abs().max().item(), "max", ref.abs().max().item())
