"""Per-atom timestamps of the sweep GEMM (debug build with -DMEC_TRACE).
Usage (GPU box): python tools/trace_sweep.py [--config C1]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C1"); ap.add_argument("--batch", type=int)
ap.add_argument("--path", default="auto"); args = ap.parse_args()
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
L.mec_sweep_trace_enable.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
assert L.mec_sweep_trace_enable(ctypes.byref(buf), ctypes.byref(nbytes)) == 0
mec.conv_forward(I, K, cfg["s_h"], cfg["s_w"], path=path); torch.cuda.synchronize()
host = np.zeros(nbytes.value // 8, dtype=np.uint64)
L.mec_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
assert L.mec_trace_read(host.ctypes.data, buf, nbytes) == 0
tr = host.reshape(160, 512, 8).astype(np.int64)
tr_rows = tr[:, 256:, :]
if os.environ.get("SW_CYCLES"):
    c = np.where(tr[:, 257, 3] > 0)[0]
    rows = tr[c][:, 257:296, :8] - 1
    print("raw", tr[c[0], 256:259, :4].tolist(), "ctas", len(c))
    rows = rows[(rows >= 0).all(axis=2)]
    print("per-row cycles (median): tempty wait %d  afull waits %d  MMA issue calls %d  row total %d  commit %d  run-loop total %d  setup %d  tail %d" % tuple(np.median(rows, axis=0)))
    sys.exit(0)
ctas = np.where(tr[:, 0, 0] > 0)[0]
t0 = tr[ctas, 0, 0].min()
life = tr[ctas, 511, :6]
ent = life[:, 0].min()
print("CTA lifetime (us after the first CTA entry), pct 0/50/100:")
for k, n in enumerate(["entry", "prologue done", "weights issued", "weights landed", "epilogue drained", "exit"]):
    v = (life[:, k] - ent) / 1e3
    print("  %-17s %7.2f %7.2f %7.2f" % (n, np.percentile(v, 0), np.percentile(v, 50), np.percentile(v, 100)))
print("  first A TMA issue %7.2f" % ((t0 - ent) / 1e3))
for c in ctas[:3]:
    print("  cta %d raw lifetime (us):" % c, " ".join("%.2f" % ((v - ent) / 1e3) for v in tr[c, 511, :6]))
pr = tr[ctas[0], 300:320, :3]
print("producer (cta %d): before-wait / after-wait / after-issue (us from t0):" % ctas[0])
for k in range(20):
    if pr[k, 0]: print("  atom %2d  %7.3f %7.3f %7.3f" % (k, (pr[k,0]-t0)/1e3, (pr[k,1]-t0)/1e3, (pr[k,2]-t0)/1e3))
names = ["P_issued", "C_full", "C_aempty", "C_arrived", "M_afull", "M_released"]
print("ctas", len(ctas))
def med(e1, e2):
    A = tr[ctas][:, :, e1]; B = tr[ctas][:, :, e2]; m = (A > 0) & (B > 0)
    return np.median((B - A)[m]) / 1e3 if m.any() else float("nan")
for c in list(ctas[:1]):
    print("cta", c, "(atoms)")
    for a in range(40):
        row = tr[c, a, :6]
        if not row.any(): break
        print("  atom %3d " % a + " ".join(f"{n}={(x - t0)/1e3:7.2f}" if x else f"{n}=   -   " for n, x in zip(names, row)))
    print("cta", c, "(rows: M tempty passed / committed)")
    for r in range(20):
        if not tr[c, r, 6]: break
        print("  row %3d  start=%7.2f  end=%7.2f  (%.2f us)" % (r, (tr[c, r, 6] - t0) / 1e3, (tr[c, r, 7] - t0) / 1e3, (tr[c, r, 7] - tr[c, r, 6]) / 1e3))
print("median us: P->C_full %.3f  C_full->C_aempty %.3f  C_aempty->C_arrived %.3f  C_arrived->M_afull %.3f" % (
    med(0, 1), med(1, 2), med(2, 3), med(3, 4)))
print("median row issue span us %.3f" % med(6, 7))
rs = tr[ctas][:, :, 6]; d = np.diff(rs, axis=1); d = d[(rs[:, 1:] > 0) & (rs[:, :-1] > 0)]
print("median us between row starts: %.3f" % (np.median(d) / 1e3))
ends = tr[ctas][:, :, :8].max(axis=(1, 2))
print("kernel span us (first TMA issue to last event): %.2f" % ((ends.max() - t0) / 1e3))
