"""Diagnostic: stage times of one conv under three L2 states before each step:
warm (no flush), dirty (a 256 MB torch fill: L2 full of dirty lines), clean
(mec.l2_flush: write then read, L2 full of clean lines)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1706_06873_b200 import mec
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
ap.add_argument("--path", type=int, default=0); ap.add_argument("--iters", type=int, default=30); args = ap.parse_args()
cfg = synth.config(args.config, args.batch)
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
I = torch.empty((cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"]), dtype=tdt, device="cuda")
K = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=tdt, device="cuda")
mec.synth_fill(I, 1, 0, 0); mec.synth_fill(K, 1, 1, 0)
s = (cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"], cfg["k_h"], cfg["k_w"], cfg["k_c"])
ws = torch.empty(mec.workspace_bytes(s, cfg["s_h"], cfg["s_w"], tdt), dtype=torch.uint8, device="cuda")
big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
O = mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], workspace=ws, path=args.path)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for e in evs: e.record()
for mode in ("warm", "dirty", "clean"):
    st = []
    for _ in range(args.iters):
        if mode == "dirty": big[: 256 << 20].fill_(np.random.randint(1, 200))
        if mode == "clean": mec.l2_flush(big)
        mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], out=O, workspace=ws, path=args.path, stage_events=evs)
        torch.cuda.synchronize()
        st.append([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(3)])
    print(args.config, mode, "lower/gemm/fix us (median):", np.median(np.array(st), axis=0).round(1), flush=True)
