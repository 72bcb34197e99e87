"""Timeline of one whole conv step (lowering + sweep GEMM) from the per-CTA
globaltimer stamps of the trace build (-DMEC_TRACE), against the CUDA-event
time of the same step.  Usage (GPU box): python tools/trace_step.py [--config C1]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
ap.add_argument("--reps", type=int, default=3); args = ap.parse_args()
from paper_1706_06873_b200 import _build, _lib
so = os.path.join(_build.ROOT, "build", "trace", "libmec_trace.so")
_build.build(extra_flags=["-DMEC_TRACE"], so_path=so, build_dir=os.path.join(_build.ROOT, "build", "trace"))
_lib.SO_PATH = so
os.environ["MEC_NO_BUILD"] = "1"
L = _lib.lib()
import torch, synth
from paper_1706_06873_b200 import mec
cfg = synth.config(args.config, args.batch)
tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
I = torch.empty((cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"]), dtype=tdt, device="cuda")
K = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=tdt, device="cuda")
mec.synth_fill(I, 1, 0, 0); mec.synth_fill(K, 1, 1, 0)
s_h, s_w = cfg["s_h"], cfg["s_w"]
ws = torch.empty(mec.workspace_bytes((cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"], cfg["k_h"], cfg["k_w"], cfg["k_c"]),
                                     s_h, s_w, tdt), dtype=torch.uint8, device="cuda")
O = mec.conv_forward(I, K, s_h, s_w, workspace=ws)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): mec.conv_forward(I, K, s_h, s_w, out=O, workspace=ws)
torch.cuda.synchronize()
bufs = {}
for name in ("lower", "sweep"):
    fn = getattr(L, f"mec_{name}_trace_enable")
    fn.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
    b = ctypes.c_void_p(); n = ctypes.c_size_t()
    assert fn(ctypes.byref(b), ctypes.byref(n)) == 0
    bufs[name] = (b, n)
L.mec_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
def read(name):
    b, n = bufs[name]
    h = np.zeros(n.value // 8, dtype=np.uint64)
    assert L.mec_trace_read(h.ctypes.data, b, n) == 0
    return h.astype(np.int64)
for rep in range(args.reps):
    mec.l2_flush(flush)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); mec.conv_forward(I, K, s_h, s_w, out=O, workspace=ws); e1.record()
    torch.cuda.synchronize()
    lo = read("lower").reshape(-1, 4)[32768:]; lo = lo[lo[:, 0] > 0]
    sw = read("sweep").reshape(160, 512, 8)[:, 511, :6]; sw = sw[sw[:, 0] > 0]
    t0 = lo[:, 0].min()
    us = lambda x: (x - t0) / 1e3
    print(f"rep {rep}: event {e0.elapsed_time(e1) * 1e3:.1f} us; lowering CTAs {len(lo)}, GEMM CTAs {len(sw)} (first 160)")
    print("  lowering: first entry 0.00, last entry %.2f, first exit %.2f, last exit %.2f" %
          (us(lo[:, 0].max()), us(lo[:, 2].min()), us(lo[:, 2].max())))
    for k, nm in enumerate(["entry", "prologue done", "weights issued", "weights landed", "epilogue drained", "exit"]):
        print("  GEMM %-17s min %7.2f  median %7.2f  max %7.2f" % (nm, us(sw[:, k].min()), us(np.median(sw[:, k])), us(sw[:, k].max())))
    print("  step span (lowering first entry -> GEMM last exit) %.2f us" % us(max(sw[:, 4].max(), sw[:, 5].max())))
