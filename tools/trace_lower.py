"""Per-CTA timeline of the lowering kernel (debug build with -DMEC_TRACE).
Usage (GPU box): python tools/trace_lower.py [--config C1]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
args = ap.parse_args()
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
mec.synth_fill(I, 1, 0, 0)
big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): Lp = mec.lower_pitched(I, cfg["k_h"], cfg["k_w"], cfg["s_h"], cfg["s_w"])
buf = ctypes.c_void_p(); nbytes = ctypes.c_size_t()
L.mec_lower_trace_enable.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
assert L.mec_lower_trace_enable(ctypes.byref(buf), ctypes.byref(nbytes)) == 0
L.mec_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
for rep in range(2):
    mec.l2_flush(big); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); mec.lower_pitched(I, cfg["k_h"], cfg["k_w"], cfg["s_h"], cfg["s_w"]); e1.record()
    torch.cuda.synchronize()
    host = np.zeros(nbytes.value // 8, dtype=np.uint64)
    assert L.mec_trace_read(host.ctypes.data, buf, nbytes) == 0
    tr = host.reshape(-1, 4).astype(np.int64)
    cta = tr[32768:]; cta = cta[cta[:, 0] > 0]
    tr = tr[:32768]
    n = int((tr[:, 0] > 0).sum()); tr = tr[:n]
    t0 = tr[:, 0].min()
    st, sg, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
    if len(cta):
        c0 = cta[:, 0].min()
        print("  CTA entry pct 0/50/100 (us from first entry): %s; first band arrival at %.2f; last CTA exit at %.2f"
              % (np.percentile((cta[:, 0] - c0) / 1e3, [0, 50, 100]).round(2), (tr[:, 0].min() - c0) / 1e3,
                 (cta[:, 2].max() - c0) / 1e3))
    print(f"rep {rep}: event {e0.elapsed_time(e1)*1e3:.1f}us  ctas {n}  span {en.max():.2f}us")
    print("  (per band) rows arrived pct 0/50/90/100: %s" % np.percentile(st, [0, 50, 90, 100]).round(2))
    print("  build dur  pct 50/90/100: %s" % np.percentile(sg - st, [50, 90, 100]).round(2))
    print("  output dur pct 50/90/100: %s" % np.percentile(en - sg, [50, 90, 100]).round(2))
    print("  written    pct 10/50/90/100: %s" % np.percentile(en, [10, 50, 90, 100]).round(2))
    sm = tr[:, 3]
    print("  bands per SM: min %d max %d" % (np.bincount(sm).min(), np.bincount(sm).max()))
