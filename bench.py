#!/usr/bin/env python
"""bench.py -- MEC hot path on B200: conv TFLOP/s + lowered bytes vs im2col.

One "step" = one pass of the whole hot path over one
batch: compact lowering (+ weight operand prep) -> window GEMMs (paper
Solution A or B by the threshold rule of Alg.2 l.8) -> Solution A's format
fix, i.e. one mec_conv_forward_ex call through the C ABI.

Default workload (N=1): BASELINE.json configs[1], AlexNet conv1 (Table 2 cv1)
I 32x227x227x3, K 11x11x3x96, stride 4, bf16.  Synthetic inputs from the
counter-based generator (synth/), generated on the device.  Multi-GPU
(torchrun, one process per GPU): each rank processes its own batch of the
same size (weak scaling; global images r*i_n .. (r+1)*i_n), K is broadcast
once from rank 0 with NCCL, no other collective on the path; time = max over
ranks of the device-timed steps.

L2 (126 MB) is flushed before every timed step (a 2x L2 write, then a 2x L2
read so the write's dirty lines are written back outside the step's CUDA events): C1's working set fits in L2.

--impl reference: the CPU oracle (oracle/, plain C fp64) timed on this box's
host cores on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv TFLOP/s (2·N·OH·OW·KH·KW·IC·KC/t) + lowered bytes vs im2col, 1/2/4/8 B200"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["mec", "reference"], default="mec")
    ap.add_argument("--config", default="C1", help="synth.configs.CONFIGS key (default C1)")
    ap.add_argument("--batch", type=int, default=None, help="override images per GPU")
    ap.add_argument("--path", choices=["auto", "A", "B", "fused"], default="auto")
    ap.add_argument("--sola-fix", choices=["epilogue", "literal"], default="epilogue")
    ap.add_argument("--T", type=int, default=100)
    ap.add_argument("--rows-per-tile", type=int, default=0,
                    help="window GEMM output rows per tile (multi-row schedule; 0 = library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4,
                    help="image chunks of the e2e host-buffer call (copies pipelined with the kernels)")
    ap.add_argument("--no-flush", action="store_true", help="(diagnostic) do not flush L2")
    ap.add_argument("--no-fused-alt", action="store_true",
                    help="with --path auto, skip measuring the fused path alongside (north_star (3))")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def workload(cfg):
    i_n, i_h, i_w, i_c = cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"]
    k_h, k_w, k_c, s_h, s_w = cfg["k_h"], cfg["k_w"], cfg["k_c"], cfg["s_h"], cfg["s_w"]
    o_h = (i_h - k_h) // s_h + 1
    o_w = (i_w - k_w) // s_w + 1
    flops = 2 * i_n * o_h * o_w * k_h * k_w * i_c * k_c
    return dict(shape=(i_n, i_h, i_w, i_c, k_h, k_w, k_c), o_h=o_h, o_w=o_w, flops=flops,
                nI=i_n * i_h * i_w * i_c, nK=k_h * k_w * i_c * k_c, nO=i_n * o_h * o_w * k_c,
                nL=i_n * o_w * i_h * k_w * i_c, nIm2col=i_n * o_h * o_w * k_h * k_w * i_c)


class ClockSampler:
    """Samples SM clock + clock-event reasons via NVML while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            self.sample_once()
            time.sleep(0.002)

    def sample_once(self):
        if not self.ok:
            return
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except AttributeError:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        if self.ok:
            self.sample_once()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self.sample_once()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline(cfg, w, dtype_name, seed):
    """The oracle (as it stands) on a bounded sample of the workload: Alg.2
    lowering + Solution-B window GEMMs in fp64, threads over images."""
    import numpy as np

    import oracle
    import synth

    cores = os.cpu_count() or 1
    kind = synth.KIND_GRID8 if dtype_name == "bf16" else synth.KIND_GRID11
    K = synth.kernel_tensor(cfg, kind, seed)
    per_img = w["flops"] / cfg["i_n"]
    # calibrate with one image on one core, then size the sample to ~10-20 s of CPU work
    I1 = synth.input_images(cfg, 0, 1, kind, seed)
    t0 = time.perf_counter()
    oracle.conv_solB(I1, K, cfg["s_h"], cfg["s_w"], n_threads=1)
    t1 = time.perf_counter() - t0
    n_img = int(max(1, min(cfg["i_n"], round(12.0 * cores / max(t1, 1e-3)))))
    n_img = max(1, min(n_img, 4 * cores, cfg["i_n"]))
    threads = min(cores, n_img)
    I = synth.input_images(cfg, 0, n_img, kind, seed)
    t0 = time.perf_counter()
    oracle.conv_solB(I, K, cfg["s_h"], cfg["s_w"], n_threads=threads)
    dt = time.perf_counter() - t0
    val = n_img * per_img / dt / 1e12
    return {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{n_img} of {cfg['i_n']} images of {cfg['name']}: oracle.conv_solB "
                      f"(Alg.2 lowering + Solution B window GEMMs, plain C, fp64), {threads} threads, "
                      f"{dt:.2f} s; the extrapolated full-batch time is {dt * cfg['i_n'] / n_img:.1f} s",
            "seconds": dt, "images": n_img, "host_cores_total": cores}


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
    import numpy as np  # noqa: F401

    import oracle
    import synth

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.config(args.config, args.batch)
    w = workload(cfg)
    seed = synth.SEED_BASE + cfg["index"]
    dtype_name = "bf16" if cfg["dtype"] == "bf16" else "tf32"
    kind = synth.KIND_GRID8 if dtype_name == "bf16" else synth.KIND_GRID11
    cores = os.cpu_count() or 1
    K = synth.kernel_tensor(cfg, kind, seed)
    per_img = w["flops"] / cfg["i_n"]
    # bounded sample per step: one image per core (at most i_n), ~1-3 s of CPU work
    I1 = synth.input_images(cfg, 0, 1, kind, seed)
    t0 = time.perf_counter()
    oracle.conv_solB(I1, K, cfg["s_h"], cfg["s_w"], n_threads=1)
    t1 = time.perf_counter() - t0
    total = args.steps + args.warmup
    budget_per_step = 150.0 / max(total, 1)  # whole run within ~2.5 minutes
    n_img = max(1, min(cfg["i_n"], cores, int(budget_per_step * cores / max(t1, 1e-3))))
    threads = min(cores, n_img)
    I = synth.input_images(cfg, 0, n_img, kind, seed)
    for _ in range(args.warmup):
        oracle.conv_solB(I, K, cfg["s_h"], cfg["s_w"], n_threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.conv_solB(I, K, cfg["s_h"], cfg["s_w"], n_threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = args.steps * n_img * per_img / tot / 1e12
    sample = (f"{n_img} of {cfg['i_n']} images of {cfg['name']} per step: oracle.conv_solB "
              f"(Alg.2 lowering + Solution B window GEMMs, plain C, fp64), {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based generator, seed %d)" % seed,
        "config": {"workload": cfg["name"], "sample_images_per_step": n_img},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import synth
    from paper_1706_06873_b200 import dist, mec
    from paper_1706_06873_b200._lib import (MEC_PATH_AUTO, MEC_PATH_FUSED, MEC_PATH_SOLUTION_A,
                                            MEC_PATH_SOLUTION_B, MEC_SOLA_FIX_EPILOGUE, MEC_SOLA_FIX_LITERAL,
                                            MecError)

    rank, ws, dev = dist.init()
    if dev.type != "cuda":
        raise SystemExit("bench.py needs CUDA GPUs (no CPU fallback)")
    cfg = synth.config(args.config, args.batch)
    w = workload(cfg)
    dtype_name = "bf16" if cfg["dtype"] == "bf16" else "tf32"
    tdt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    elt = 2 if dtype_name == "bf16" else 4
    kind = synth.KIND_GRID8 if dtype_name == "bf16" else synth.KIND_GRID11
    seed = synth.SEED_BASE + cfg["index"]
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = w["shape"]
    s_h, s_w = cfg["s_h"], cfg["s_w"]
    path = {"auto": MEC_PATH_AUTO, "A": MEC_PATH_SOLUTION_A, "B": MEC_PATH_SOLUTION_B,
            "fused": MEC_PATH_FUSED}[args.path]
    fix = MEC_SOLA_FIX_EPILOGUE if args.sola_fix == "epilogue" else MEC_SOLA_FIX_LITERAL

    # ---- inputs: this rank's images (global index offset), K from rank 0 by NCCL broadcast
    I = torch.empty((i_n, i_h, i_w, i_c), dtype=tdt, device=dev)
    mec.synth_fill(I, seed, synth.TENSOR_I, kind, index_offset=rank * i_n * i_h * i_w * i_c)
    K = torch.empty((k_h, k_w, i_c, k_c), dtype=tdt, device=dev)
    if rank == 0:
        mec.synth_fill(K, seed, synth.TENSOR_K, kind)
    dist.broadcast_weights(K, 0)
    K_local = torch.empty_like(K)
    mec.synth_fill(K_local, seed, synth.TENSOR_K, kind)
    k_bcast_ok = bool(torch.equal(K, K_local))
    del K_local
    O = torch.empty((i_n, w["o_h"], w["o_w"], k_c), dtype=tdt, device=dev)
    ws_bytes = mec.workspace_bytes(w["shape"], s_h, s_w, tdt)
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(4 * l2, 128 << 20), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        return mec.conv_forward(I, K, s_h, s_w, out=O, path=path, T=args.T, sola_fix=fix, rows_per_tile=args.rows_per_tile,
                                workspace=workspace, stage_events=evs, return_path=True)

    # ---- memory: device-memory delta of one pooled call (library allocates L itself)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(dev)[0]
    mec.conv_forward(I, K, s_h, s_w, out=O, path=path, T=args.T, sola_fix=fix, rows_per_tile=args.rows_per_tile)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(dev)[0]
    pooled_delta = max(0, free0 - free1)

    # ---- warm-up
    for _ in range(max(args.warmup, 0)):
        if not args.no_flush:
            mec.l2_flush(flush)
        _, chosen = step()
    torch.cuda.synchronize()
    launches_per_step = mec.last_launch_count()

    # ---- timed region: K steps, CUDA events on the launching stream around each
    # step only (events between the step's kernels would serialise the window
    # GEMM's programmatic dependent launch)
    K_steps = args.steps
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K_steps)]
    sampler = ClockSampler(dev.index)
    dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for k in range(K_steps):
            if not args.no_flush:
                mec.l2_flush(flush)
            sev[k][0].record()
            step()
            sev[k][1].record()
        torch.cuda.synchronize()
    dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in sev]
    tot_ms = dist.max_over_ranks(sum(step_ms), dev)
    value = w["flops"] * ws * K_steps / (tot_ms * 1e-3) / 1e12

    # ---- per-kernel times (roofline): K more steps with the library's stage
    # events between the kernels (kernels serialised, so each is timed alone)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K_steps)]
    for e4 in evs:  # torch creates events lazily: create them now; the library re-records them
        for e in e4:
            e.record()
    torch.cuda.synchronize()
    for k in range(K_steps):
        if not args.no_flush:
            mec.l2_flush(flush)
        step(evs[k])
    torch.cuda.synchronize()
    lower_ms = [e[0].elapsed_time(e[1]) for e in evs]
    gemm_ms = [e[1].elapsed_time(e[2]) for e in evs]
    fix_ms = [e[2].elapsed_time(e[3]) for e in evs]

    # ---- CUDA-graph replay of the same step (launch gaps removed), diagnostic
    graph_ms = None
    try:
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream(dev)
        s2.wait_stream(stream)
        with torch.cuda.stream(s2):
            step()
            with torch.cuda.graph(g, stream=s2):
                step()
        stream.wait_stream(s2)
        torch.cuda.synchronize()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K_steps)]
        for a, b in gev:
            if not args.no_flush:
                mec.l2_flush(flush)
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        graph_ms = statistics.mean(a.elapsed_time(b) for a, b in gev)
    except Exception as e:  # noqa: BLE001
        graph_ms = f"unavailable: {e}"

    # ---- end to end through the public API with host buffers (pinned), copies timed:
    # mec_conv_forward_host copies I and K in and O out inside the call, pipelined over
    # image chunks on three streams (the copies of neighbouring chunks overlap the kernels)
    e2e = None
    if not args.no_e2e:
        I_h = I.cpu().pin_memory()
        K_h = K.cpu().pin_memory()
        O_h = torch.empty(O.shape, dtype=O.dtype).pin_memory()
        nch = max(1, min(args.e2e_chunks, I.shape[0]))
        scratch = torch.empty(mec.host_scratch_bytes(*I.shape, *K.shape[:2], K.shape[3], s_h, s_w, I.dtype, nch),
                              dtype=torch.uint8, device=dev)
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K_steps)]

        def e2e_call():
            mec.conv_forward_host(I_h, K_h, s_h, s_w, out=O_h, n_chunks=nch, path=path, T=args.T,
                                  sola_fix=fix, scratch=scratch)

        for _ in range(2):
            e2e_call()
        dist.barrier()
        torch.cuda.synchronize()
        e2e_launches = 0
        for a, b in eev:
            if not args.no_flush:
                mec.l2_flush(flush)
            a.record()
            e2e_call()
            e2e_launches += mec.last_launch_count()
            b.record()
        torch.cuda.synchronize()
        dist.barrier()
        e2e_ms = dist.max_over_ranks(sum(a.elapsed_time(b) for a, b in eev), dev)
        e2e = {"value": w["flops"] * ws * K_steps / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": (w["nI"] + w["nK"]) * elt, "d2h_bytes_per_step": w["nO"] * elt,
               "ms_per_step": e2e_ms / K_steps, "api": "mec_conv_forward_host",
               "chunks": nch, "kernels_per_step": e2e_launches / K_steps}

    # ---- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    mean_lower = statistics.mean(lower_ms)
    mean_gemm = statistics.mean(gemm_ms)
    mean_fix = statistics.mean(fix_ms)
    fused = chosen == MEC_PATH_FUSED
    bytes_lower = (w["nI"] + w["nL"]) * elt                 # read I, write L
    bytes_gemm = (w["nL"] + w["nK"] + w["nO"]) * elt        # L read once, K, write O
    if fused:  # (a6): no L; the GEMM reads I (windows) and K, writes O
        bytes_lower = (w["nK"] * 2) * elt                   # weight operand prep: read K, write Kt
        bytes_gemm = (w["nI"] + w["nK"] + w["nO"]) * elt
    flops = w["flops"]
    hbm = peaks["hbm_gbs"]
    tc = peaks["bf16_tflops"] if dtype_name == "bf16" else peaks["bf16_tflops"] / 2.0
    tc_src = "bf16 measured burst" if dtype_name == "bf16" else "tf32 = bf16 measured burst x 1/2 (nominal ratio)"
    kernels = {
        ("weight_prep" if fused else "mec_lower"): (mean_lower, "hbm", bytes_lower / (mean_lower * 1e-3) / 1e9,
                                                    hbm, "GB/s", bytes_lower),
    }
    t_mem, t_tc = bytes_gemm / (hbm * 1e9), flops / (tc * 1e12)
    gname = "fused_window_gemm" if fused else "window_gemm"
    if t_mem >= t_tc:
        kernels[gname] = (mean_gemm, "hbm", bytes_gemm / (mean_gemm * 1e-3) / 1e9, hbm, "GB/s", bytes_gemm)
    else:
        kernels[gname] = (mean_gemm, "tensor", flops / (mean_gemm * 1e-3) / 1e12, tc, "TFLOP/s", flops)
    if chosen == MEC_PATH_SOLUTION_A and fix == MEC_SOLA_FIX_LITERAL:
        bfix = 4 * w["nO"] * elt
        kernels["sola_format_fix"] = (mean_fix, "hbm", bfix / (mean_fix * 1e-3) / 1e9, hbm, "GB/s", bfix)
    dom = max(kernels, key=lambda k: kernels[k][0])
    ms, bound, ach, peak, unit, alg = kernels[dom]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(cfg["name"], {}).get(dom)
    roof = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
            "traffic": traffic, "kernel": dom, "kernel_ms": ms, "algorithmic_per_launch": alg,
            "peak_source": peak_src if bound == "hbm" else f"{tc_src} ({peak_src})",
            "all_kernels": {k: {"ms": v[0], "bound": v[1], "achieved": v[2], "unit": v[4],
                                "frac": v[2] / v[3]} for k, v in kernels.items()}}

    # ---- north_star (3): the optional fused path measured against the two-kernel
    # path, same workload, same timing rules (reported alongside; `value` stays the
    # paper's path of Alg.2 l.8)
    fused_alt = None
    if args.path == "auto" and not args.no_fused_alt:
        def fstep(evs=None):
            return mec.conv_forward(I, K, s_h, s_w, out=O, path=MEC_PATH_FUSED, workspace=workspace,
                                    stage_events=evs, return_path=True)
        try:
            for _ in range(max(args.warmup, 0)):
                if not args.no_flush:
                    mec.l2_flush(flush)
                fstep()
            fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(K_steps)]
            torch.cuda.synchronize()
            for a, b in fev:
                if not args.no_flush:
                    mec.l2_flush(flush)
                a.record()
                fstep()
                b.record()
            torch.cuda.synchronize()
            f_tot = dist.max_over_ranks(sum(a.elapsed_time(b) for a, b in fev), dev)
            fse = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K_steps)]
            for e4 in fse:
                for e in e4:
                    e.record()
            torch.cuda.synchronize()
            for k in range(K_steps):
                if not args.no_flush:
                    mec.l2_flush(flush)
                fstep(fse[k])
            torch.cuda.synchronize()
            f_prep = statistics.mean(e[0].elapsed_time(e[1]) for e in fse)
            f_gemm = statistics.mean(e[1].elapsed_time(e[2]) for e in fse)
            fb = (w["nI"] + w["nK"] + w["nO"]) * elt
            if fb / (hbm * 1e9) >= flops / (tc * 1e12):
                f_roof = {"kernel": "fused_window_gemm", "bound": "hbm", "unit": "GB/s",
                          "achieved": fb / (f_gemm * 1e-3) / 1e9, "peak": hbm}
            else:
                f_roof = {"kernel": "fused_window_gemm", "bound": "tensor", "unit": "TFLOP/s",
                          "achieved": flops / (f_gemm * 1e-3) / 1e12, "peak": tc}
            f_roof["frac"] = f_roof["achieved"] / f_roof["peak"]
            fused_alt = {"path": "fused_lowering_in_gemm",
                         "value": w["flops"] * ws * K_steps / (f_tot * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "ms_per_step": f_tot / K_steps,
                         "stages_ms": {"weight_prep": f_prep, "fused_window_gemm": f_gemm},
                         "roofline": f_roof, "gpu_launches": mec.last_launch_count() * K_steps}
        except MecError as e:
            fused_alt = {"path": "fused_lowering_in_gemm", "unavailable": str(e)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, w, dtype_name, seed)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}

    names = {MEC_PATH_SOLUTION_A: "solution_A_batch_folded", MEC_PATH_SOLUTION_B: "solution_B_per_image",
             MEC_PATH_FUSED: "fused_lowering_in_gemm"}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": K_steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / K_steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dtype_name,
        "data": f"synthetic (counter-based generator on device, seed {seed}, GRID values exact in {dtype_name})",
        "config": {
            "workload": cfg["name"], "i_n_per_gpu": i_n, "global_batch": i_n * ws,
            "I": [i_n, i_h, i_w, i_c], "K": [k_h, k_w, i_c, k_c], "stride": [s_h, s_w],
            "O": [i_n, w["o_h"], w["o_w"], k_c],
            "path": names.get(chosen, str(chosen)),
            "path_rule": f"Alg.2 l.8: Solution A iff o_w <= T={args.T} and #O <= #L" if path == MEC_PATH_AUTO
            else "forced",
            "north_star_letter": "B" if chosen == MEC_PATH_SOLUTION_A else "A",
            "sola_fix": args.sola_fix if chosen == MEC_PATH_SOLUTION_A else None,
            "rows_per_tile": args.rows_per_tile or 1,
            "l2": "flushed before every timed step: a 2x L2 write, then a 2x L2 read that writes its dirty lines back (outside the timed region)" if not args.no_flush else "warm (not flushed)",
            "parallelism": f"dp{ws} (images sharded per GPU, K broadcast once by NCCL)",
        },
        "lowered_bytes": {
            "mec_L": w["nL"] * elt, "im2col_L": w["nIm2col"] * elt,
            "im2col_over_mec": w["nIm2col"] / w["nL"], "workspace_allocated": ws_bytes,
            "pooled_call_device_mem_delta": pooled_delta,
        },
        "stages_ms": {"lower": mean_lower, "gemm": mean_gemm, "format_fix": mean_fix},
        "stages_timing": "per-kernel CUDA events in a separate run of K steps (kernels serialised); "
                         "value / ms_per_step time whole steps with no events inside them",
        "graph_ms_per_step": graph_ms,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "fused_path": fused_alt,
        "gpu_launches": launches_per_step * K_steps,
        "gpu_launches_detail": {"per_step": launches_per_step, "l2_flush_kernels": 0 if args.no_flush else 2 * K_steps},
        "clocks": sampler.summary(),
        "k_broadcast_verified": k_bcast_ok,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
