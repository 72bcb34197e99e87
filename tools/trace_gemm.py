"""Per-tile stage timestamps of the window GEMM (debug build with -DMEC_TRACE).
Usage (GPU box): python tools/trace_gemm.py [--config C1] [--path A]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
ap.add_argument("--path", default="auto"); ap.add_argument("--quiet", action="store_true"); args = ap.parse_args()
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
path = {"auto": 0, "A": 1, "B": 2, "fused": 3}[args.path]
for _ in range(3): mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], path=path)
torch.cuda.synchronize()
buf = ctypes.c_void_p(); nbytes = ctypes.c_size_t()
L.mec_trace_enable.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
assert L.mec_trace_enable(ctypes.byref(buf), ctypes.byref(nbytes)) == 0
mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], path=path); torch.cuda.synchronize()
host = np.zeros(nbytes.value // 8, dtype=np.uint64)
L.mec_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
assert L.mec_trace_read(host.ctypes.data, buf, nbytes) == 0
tr = host.reshape(1024, 64, 16).astype(np.int64)
ctas = np.where(tr[:512, 0, 7] > 0)[0]
t0 = tr[ctas, 0, 7].min()
names = ["P_start", "P_issued", "M_tempty", "M_full0", "M_commit", "E_tfull", "E_done"]
print("ctas", len(ctas), "MEC_DEBUG_FLAGS", os.environ.get("MEC_DEBUG_FLAGS"))
for c in ([] if args.quiet else list(ctas[:2]) + [ctas[-1]]):
    print(f"cta {c}: start {(tr[c,0,7]-t0)/1e3:.2f}us")
    for tl in range(64):
        row = tr[c, tl, :7]
        if row[0] == 0 and row[2] == 0: break
        extra = "".join(f" {n}={(tr[c, tl, e] - t0)/1e3:7.2f}" for n, e in
                        (("R_wait", 7), ("R_dec", 8), ("R_arm", 9), ("R_cp0", 10), ("R_cp1", 11), ("R_req", 15))
                        if tr[c, tl, e])
        print("  tile", tl, " ".join(f"{n}={(x - t0)/1e3:7.2f}" if x else f"{n}=   -   " for n, x in zip(names, row)) + extra)
# SM clock: clock64 / globaltimer deltas over each CTA's lifetime (slot 62)
ck = tr[ctas, 62, :4]
ok = (ck[:, 3] > ck[:, 2])
if ok.any():
    mhz = (ck[ok, 1] - ck[ok, 0]) / ((ck[ok, 3] - ck[ok, 2]) / 1e3) 
    print("SM clock over CTA lifetimes (MHz): median %.0f min %.0f max %.0f" % (np.median(mhz), mhz.min(), mhz.max()))
# aggregates
ends = tr[ctas][:, :, 6]; ends = ends[ends > 0]
print("kernel span us", (ends.max() - t0) / 1e3)
mma = (tr[ctas][:, :, 4] - tr[ctas][:, :, 3]); mma = mma[(tr[ctas][:, :, 4] > 0) & (tr[ctas][:, :, 3] > 0)]
epi = (tr[ctas][:, :, 6] - tr[ctas][:, :, 5]); epi = epi[(tr[ctas][:, :, 6] > 0) & (tr[ctas][:, :, 5] > 0)]
wait_full = (tr[ctas][:, :, 3] - tr[ctas][:, :, 2]); wait_full = wait_full[(tr[ctas][:, :, 3] > 0) & (tr[ctas][:, :, 2] > 0)]
print("per-tile MMA issue span us: median %.2f" % (np.median(mma) / 1e3))
print("per-tile epilogue us: median %.2f" % (np.median(epi) / 1e3))
print("per-tile wait first full after tempty us: median %.2f" % (np.median(wait_full) / 1e3))
sub = tr[ctas][:, 1:, :]
def med(a, b):
    m = (sub[:, :, a] > 0) & (sub[:, :, b] > 0)
    return np.median((sub[:, :, b] - sub[:, :, a])[m]) / 1e3 if m.any() else float('nan')
if (sub[:, :, 15] > 0).any():
    print("gather: rempty->copies issued %.3f | copies issued->rows ready %.3f | rows ready->built %.3f" % (
        med(7, 15), med(15, 0), med(0, 1)))
    print("gather: built(t-2) -> rempty(t) passed %.3f" % np.median(((sub[:, 2:, 7] - sub[:, :-2, 1]))[(sub[:, 2:, 7] > 0) & (sub[:, :-2, 1] > 0)] / 1e3))
b2 = tr[512 + ctas][:, 1:, :]
if (b2[:, :, 0] > 0).any():
    def med2(bank_a, ia, bank_b, ib):
        A = bank_a[:, :, ia]; B = bank_b[:, :, ib]; m = (A > 0) & (B > 0)
        return np.median((B - A)[m]) / 1e3 if m.any() else float('nan')
    for q in range(4):
        print(f"builder quarter {q} full arrived (us after M_tempty), atoms 0-3:",
              " ".join("%.2f" % med2(sub, 2, b2, q * 4 + k) for k in range(4)))
if (sub[:, :, 14] > 0).any():
    print("gather MMA full-wait passes (us after tempty), median per atom:",
          " ".join("%.2f" % med(2, 8 + k) for k in range(7)))
    print("stages", os.environ.get("MEC_DEBUG_STAGES"))
print("epilogue breakdown (median us, tiles >= 1): tfull->p0 ldwait %.3f | ldwait->bulkwait %.3f | bulkwait->staged %.3f | p0 staged->p1 ldwait %.3f | p1 ldwait->bulkwait %.3f | p1 bulkwait->staged %.3f | p1 staged -> done %.3f" % (
    med(5, 8), med(8, 10), med(10, 9), med(9, 12), med(12, 14), med(14, 13), med(13, 6)))
