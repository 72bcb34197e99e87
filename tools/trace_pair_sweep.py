"""Cycle accounting of the CTA-pair atom-major sweep (debug build with -DMEC_TRACE):
per CTA the MMA warp's cycles waiting for a free accumulator and for landed
atoms, and the producer's cycles waiting for a free stage.
Usage (GPU box): python tools/trace_pair_sweep.py --config C4_cv4 --batch 128"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C4_cv4"); ap.add_argument("--batch", type=int)
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
K = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=tdt, device="cuda")
mec.synth_fill(I, 1, 0, 0); mec.synth_fill(K, 1, 1, 0)
O, g = mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], return_gemm=True)
assert g == 4, f"the pair sweep did not run (kernel {g})"
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = ctypes.c_void_p(); nbytes = ctypes.c_size_t()
L.mec_pair_sweep_trace_enable.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
assert L.mec_pair_sweep_trace_enable(ctypes.byref(buf), ctypes.byref(nbytes)) == 0
L.mec_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
for rep in range(2):
    mec.l2_flush(flush)
    mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], out=O)
    torch.cuda.synchronize()
h = np.zeros(nbytes.value // 8, dtype=np.uint64)
assert L.mec_trace_read(h.ctypes.data, buf, nbytes) == 0
t = h.reshape(512, 8).astype(np.int64)
mma = t[t[:, 2] > 0]; prod = t[t[:, 4] > 0]
print(f"{args.config}: {len(mma)} leader MMA warps, {len(prod)} producers")
print("MMA warp: total %.0f cyc; waiting for a free accumulator %.1f%%, for landed atoms %.1f%% (medians)" % (
    np.median(mma[:, 2]), 100 * np.median(mma[:, 0] / mma[:, 2]), 100 * np.median(mma[:, 1] / mma[:, 2])))
print("producer: total %.0f cyc; waiting for a free stage %.1f%%; atoms %d; cycles per atom %.0f" % (
    np.median(prod[:, 4]), 100 * np.median(prod[:, 3] / prod[:, 4]), np.median(prod[:, 5]),
    np.median(prod[:, 4] / np.maximum(prod[:, 5], 1))))
print("rows per MMA warp (median) %d; MMA total pct 10/50/90: %s" % (
    np.median(mma[:, 6]), np.percentile(mma[:, 2], [10, 50, 90]).round()))
