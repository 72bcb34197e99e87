"""Stage micro-timing: lowering / GEMM / whole conv, warm vs L2-flushed (diagnostic)."""
import argparse, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1706_06873_b200 import mec
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
ap.add_argument("--iters", type=int, default=50); args = ap.parse_args()
cfg = synth.config(args.config, args.batch)
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
I = torch.empty((cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"]), dtype=tdt, device="cuda")
K = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=tdt, device="cuda")
mec.synth_fill(I, 1, 0, 0); mec.synth_fill(K, 1, 1, 0)
s = (cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"], cfg["k_h"], cfg["k_w"], cfg["k_c"])
ws = torch.empty(mec.workspace_bytes(s, cfg["s_h"], cfg["s_w"], tdt), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
O = mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], workspace=ws)
def t(fn, flush_first):
    res = []
    for _ in range(args.iters):
        if flush_first: mec.l2_flush(flush)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize(); res.append(a.elapsed_time(b) * 1e3)
    return statistics.median(res)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for e in evs: e.record()
def conv(): mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], out=O, workspace=ws)
def conv_ev(): mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], out=O, workspace=ws, stage_events=evs)
Ld = torch.empty((cfg["i_n"], (cfg["i_w"]-cfg["k_w"])//cfg["s_w"]+1, cfg["i_h"], cfg["k_w"], cfg["i_c"]), dtype=tdt, device="cuda")
def low(): mec.lower(I, cfg["k_h"], cfg["k_w"], cfg["s_h"], cfg["s_w"], out=Ld)
for fl in (False, True):
    print(f"flush={fl}: conv {t(conv, fl):.1f}us  mec_lower(dense) {t(low, fl):.1f}us")
    st = []
    for _ in range(args.iters):
        if fl: mec.l2_flush(flush)
        conv_ev(); torch.cuda.synchronize()
        st.append([evs[i].elapsed_time(evs[i+1]) * 1e3 for i in range(3)])
    import numpy as np
    print("   stages lower/gemm/fix (median us):", np.median(np.array(st), axis=0).round(1))
