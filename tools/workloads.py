"""Measurement harness for SURVEY.md section 8(f) NEXT rows (one B200).

  python tools/workloads.py resnet101 [--batch 32]   # NEXT-1: Table 3 weighted workload
  python tools/workloads.py stride    [--batch 32]   # NEXT-2: cv1, s = 1..10 (Fig. 4(a))
  python tools/workloads.py paths     [--batch 128]  # NEXT-3: Solution A vs B vs fused per layer
  python tools/workloads.py next4     [--batch 32]   # NEXT-4: pool consumer of h-n-w-c; virtual padding

Every conv goes through the C ABI (mec_conv_forward_ex) on device-generated
synthetic inputs; each timed call is preceded by an L2 flush outside its CUDA
events; the median of --steps calls is reported.  Memory columns are the
closed forms of Table 1 / Eq. 2 (#L_MEC, #L_im2col), the sizes the library
actually allocates (mec_workspace_bytes) and, for NEXT-1, Table 3's own
units (fp32, one image, MiB: DESIGN.md readings Q1 and Q16).
Results: one JSON line per measurement on stdout, and the whole run in
profiles/r1_next_<mode>.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1706_06873_b200 import mec  # noqa: E402
from paper_1706_06873_b200._lib import (MEC_PATH_AUTO, MEC_PATH_FUSED, MEC_PATH_SOLUTION_A,  # noqa: E402
                                        MEC_PATH_SOLUTION_B, MEC_SOLA_FIX_EPILOGUE, MEC_SOLA_FIX_LITERAL,
                                        MEC_SOLA_FIX_NONE, MecError)

PATHS = {"auto": MEC_PATH_AUTO, "A": MEC_PATH_SOLUTION_A, "B": MEC_PATH_SOLUTION_B, "fused": MEC_PATH_FUSED}
NAMES = {MEC_PATH_SOLUTION_A: "A", MEC_PATH_SOLUTION_B: "B", MEC_PATH_FUSED: "fused"}
# Table 3: ResNet-101 layers and how often each occurs
RESNET101 = [("cv4", 1), ("cv9", 3), ("cv10", 4), ("cv11", 23), ("cv12", 3)]


def dims(shape, s):
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
    return (i_h - k_h) // s + 1, (i_w - k_w) // s + 1


def flops(shape, s):
    o_h, o_w = dims(shape, s)
    i_n, _, _, i_c, k_h, k_w, k_c = shape
    return 2.0 * i_n * o_h * o_w * k_h * k_w * i_c * k_c


class Timer:
    def __init__(self, steps, warmup):
        self.steps, self.warmup = steps, warmup
        self.flush = torch.empty(4 * 126 * 2 ** 20, dtype=torch.uint8, device="cuda")

    def conv(self, shape, s, dtype, path):
        """Median device ms of one mec_conv_forward_ex call, and the path that ran."""
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
        o_h, o_w = dims(shape, s)
        I = torch.empty((i_n, i_h, i_w, i_c), dtype=tdt, device="cuda")
        K = torch.empty((k_h, k_w, i_c, k_c), dtype=tdt, device="cuda")
        mec.synth_fill(I, 1, synth.TENSOR_I, synth.KIND_GRID8)
        mec.synth_fill(K, 1, synth.TENSOR_K, synth.KIND_GRID8)
        O = torch.empty((i_n, o_h, o_w, k_c), dtype=tdt, device="cuda")
        ws = torch.empty(mec.workspace_bytes(shape, s, s, tdt), dtype=torch.uint8, device="cuda")
        chosen = None
        for _ in range(self.warmup):
            _, chosen = mec.conv_forward(I, K, s, s, out=O, path=PATHS[path], workspace=ws, return_path=True)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(self.steps)]
        for a, b in ev:
            mec.l2_flush(self.flush)
            a.record()
            mec.conv_forward(I, K, s, s, out=O, path=PATHS[path], workspace=ws)
            b.record()
        torch.cuda.synchronize()
        del I, K, O, ws
        return statistics.median(a.elapsed_time(b) for a, b in ev), NAMES.get(chosen, str(chosen))


def memory(shape, s, elt):
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
    o_h, o_w = dims(shape, s)
    n_l = i_n * o_w * i_h * k_w * i_c          # Table 1 / Alg.2 l.2
    n_im2col = i_n * o_h * o_w * k_h * k_w * i_c  # Eq. 2 with i_c
    return {"L_mec_bytes": n_l * elt, "L_im2col_bytes": n_im2col * elt,
            "ratio_im2col_over_mec": n_im2col / n_l,
            "workspace_bytes": mec.workspace_bytes(shape, s, s, torch.bfloat16 if elt == 2 else torch.float32)}


def try_conv(tm, shape, s, dtype, path):
    try:
        return tm.conv(shape, s, dtype, path)
    except MecError as e:
        return None, f"unsupported ({e})"


def resnet101(args, tm):
    rows, tot = [], {"auto": 0.0, "best": 0.0, "mem_mec_fp32_b1": 0.0, "mem_im2col_fp32_b1": 0.0}
    for name, weight in RESNET101:
        i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
        shape = (args.batch, i_h, i_w, i_c, k_h, k_w, k_c)
        t_auto, p_auto = tm.conv(shape, s, "bf16", "auto")
        t_fused, _ = try_conv(tm, shape, s, "bf16", "fused")
        best = min(t for t in (t_auto, t_fused) if t is not None)
        m1 = memory((1, i_h, i_w, i_c, k_h, k_w, k_c), s, 4)  # Table 3's units: fp32, one image
        row = {"layer": name, "weight": weight, "batch": args.batch, "dtype": "bf16", "path_auto": p_auto,
               "ms_auto": t_auto, "ms_fused": t_fused, "ms_best": best,
               "tflops_best": flops(shape, s) / (best * 1e-3) / 1e12,
               "mem_mec_MiB_fp32_b1": m1["L_mec_bytes"] / 2 ** 20,
               "mem_im2col_MiB_fp32_b1": m1["L_im2col_bytes"] / 2 ** 20,
               "memory_at_batch": memory(shape, s, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        tot["auto"] += weight * t_auto
        tot["best"] += weight * best
        tot["mem_mec_fp32_b1"] += weight * row["mem_mec_MiB_fp32_b1"]
        tot["mem_im2col_fp32_b1"] += weight * row["mem_im2col_MiB_fp32_b1"]
    summary = {"workload": "ResNet-101 weighted (Table 3 weights 1,3,4,23,3)", "batch": args.batch,
               "weighted_ms_auto": tot["auto"], "weighted_ms_best": tot["best"],
               "weighted_mem_MiB_mec_fp32_b1": tot["mem_mec_fp32_b1"],
               "weighted_mem_MiB_im2col_fp32_b1": tot["mem_im2col_fp32_b1"],
               "memory_ratio_im2col_over_mec": tot["mem_im2col_fp32_b1"] / tot["mem_mec_fp32_b1"],
               "paper_table3_mobile": {"mem_MiB_conv": 203.6, "mem_MiB_mec": 64.6, "ms_conv": 1701.6, "ms_mec": 1391.6,
                                       "hardware": "ARM7 MSM8960, batch 1 (context, not the target)"}}
    print(json.dumps(summary), flush=True)
    return {"rows": rows, "summary": summary}


def stride(args, tm):
    i_h, i_w, i_c, k_h, k_w, k_c, _ = synth.TABLE2["cv1"]
    rows = []
    for s in range(1, 11):
        shape = (args.batch, i_h, i_w, i_c, k_h, k_w, k_c)
        t_auto, p_auto = tm.conv(shape, s, "bf16", "auto")
        t_fused, _ = try_conv(tm, shape, s, "bf16", "fused")
        row = {"layer": "cv1", "s": s, "k_over_s": k_h / s, "batch": args.batch, "path_auto": p_auto,
               "ms_auto": t_auto, "ms_fused": t_fused,
               "tflops_auto": flops(shape, s) / (t_auto * 1e-3) / 1e12,
               "tflops_fused": flops(shape, s) / (t_fused * 1e-3) / 1e12 if t_fused else None,
               **memory(shape, s, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return {"rows": rows}


def paths(args, tm):
    rows = []
    for name in [f"cv{i}" for i in range(1, 13)]:
        i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
        shape = (args.batch, i_h, i_w, i_c, k_h, k_w, k_c)
        o_h, o_w = dims(shape, s)
        row = {"layer": name, "batch": args.batch, "o_w": o_w, "o_h": o_h, "k_c": k_c,
               "O_le_L": o_h * k_c <= i_h * k_w * i_c}
        for p in ("A", "B", "fused"):
            t, _ = try_conv(tm, shape, s, "bf16", p)
            row["ms_" + p] = t
        t_ab = {p: row["ms_" + p] for p in ("A", "B") if row["ms_" + p] is not None}
        row["faster_of_A_B"] = min(t_ab, key=t_ab.get) if t_ab else None
        row["paper_rule_T100"] = "A" if (o_w <= 100 and row["O_le_L"]) else "B"
        rows.append(row)
        print(json.dumps(row), flush=True)
    return {"rows": rows}


def timed(tm, fn):
    """Median device ms of fn() (L2 flushed before each call, outside the events)."""
    for _ in range(tm.warmup):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(tm.steps)]
    for a, b in ev:
        mec.l2_flush(tm.flush)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def next4(args, tm):
    rows = []
    # (1) AlexNet conv1 -> pool1 (3x3, stride 2): Solution A's output consumed by pooling
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2["cv1"]
    shape = (args.batch, i_h, i_w, i_c, k_h, k_w, k_c)
    o_h, o_w = dims(shape, s)
    I = torch.empty(shape[:4], dtype=torch.bfloat16, device="cuda")
    K = torch.empty((k_h, k_w, i_c, k_c), dtype=torch.bfloat16, device="cuda")
    mec.synth_fill(I, 1, synth.TENSOR_I, synth.KIND_GRID8)
    mec.synth_fill(K, 1, synth.TENSOR_K, synth.KIND_GRID8)
    O = torch.empty((args.batch, o_h, o_w, k_c), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(mec.workspace_bytes(shape, s, s, torch.bfloat16), dtype=torch.uint8, device="cuda")
    variants = {
        "literal_fix_then_pool": (MEC_SOLA_FIX_LITERAL, False),   # the paper's Alg.2 l.13-19, then pool
        "epilogue_fix_then_pool": (MEC_SOLA_FIX_EPILOGUE, False), # permutation in the GEMM epilogue
        "hnwc_pool_no_fix": (MEC_SOLA_FIX_NONE, True),            # pool consumes h-n-w-c
    }
    for name, (fix, hnwc) in variants.items():
        def step(fix=fix, hnwc=hnwc):
            mec.conv_forward(I, K, s, s, out=O, path=MEC_PATH_SOLUTION_A, sola_fix=fix, workspace=ws)
            X = O.view(o_h, args.batch, o_w, k_c) if hnwc else O
            mec.maxpool(X, 3, 3, 2, 2, hnwc=hnwc)
        row = {"case": "cv1 + maxpool 3x3/2", "variant": name, "batch": args.batch, "ms": timed(tm, step)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    del I, K, O, ws
    # (2) ResNet-50 conv1: 224x224x3, 7x7 stride 2, pad 3, 64 filters -- virtual padding vs a
    # materialised padded copy of I
    shape = (args.batch, 224, 224, 3, 7, 7, 64)
    I = torch.empty(shape[:4], dtype=torch.bfloat16, device="cuda")
    K = torch.empty((7, 7, 3, 64), dtype=torch.bfloat16, device="cuda")
    mec.synth_fill(I, 1, synth.TENSOR_I, synth.KIND_GRID8)
    mec.synth_fill(K, 1, synth.TENSOR_K, synth.KIND_GRID8)
    o = (224 + 6 - 7) // 2 + 1
    O = torch.empty((args.batch, o, o, 64), dtype=torch.bfloat16, device="cuda")
    Ip = torch.zeros((args.batch, 230, 230, 3), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(mec.workspace_bytes((args.batch, 230, 230, 3, 7, 7, 64), 2, 2, torch.bfloat16),
                     dtype=torch.uint8, device="cuda")

    def virtual():
        mec.conv_forward(I, K, 2, 2, out=O, workspace=ws, pad_h=3, pad_w=3)

    def materialised():
        Ip[:, 3:227, 3:227, :].copy_(I)  # the padded copy the paper assumes (border stays zero)
        mec.conv_forward(Ip, K, 2, 2, out=O, workspace=ws)

    for name, fn in (("virtual_padding", virtual), ("materialised_padded_copy", materialised)):
        row = {"case": "ResNet-50 conv1 224x224x3 7x7/2 pad 3", "variant": name, "batch": args.batch,
               "ms": timed(tm, fn),
               "extra_bytes": 0 if name == "virtual_padding" else Ip.numel() * 2}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return {"rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["resnet101", "stride", "paths", "next4"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.batch is None:
        args.batch = 128 if args.mode == "paths" else 32
    tm = Timer(args.steps, args.warmup)
    res = {"resnet101": resnet101, "stride": stride, "paths": paths, "next4": next4}[args.mode](args, tm)
    res["gpu"] = torch.cuda.get_device_name(0)
    out = args.out or os.path.join(ROOT, "gpurun_out", f"r1_next_{args.mode}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
