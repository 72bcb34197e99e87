import sys, os; sys.path.insert(0, os.getcwd())
import torch, synth, numpy as np
from paper_1706_06873_b200 import mec
for b in (2, 4, 32):
    I = torch.randn(b, 227, 227, 3, device="cuda").bfloat16(); K = torch.randn(11, 11, 3, 96, device="cuda").bfloat16()
    for fn in ("lower_pitched", "conv"):
        try:
            if fn == "conv": mec.conv_forward(I, K, 4, 4)
            else: mec.lower_pitched(I, 11, 11, 4, 4)
            torch.cuda.synchronize(); print(b, fn, "ok")
        except Exception as e: print(b, fn, "ERR", e)
