#!/usr/bin/env python
"""bench.py -- MEC hot path on B200: conv TFLOP/s + lowered bytes vs im2col.

One "step" = one pass of the whole hot path over one
batch: compact lowering (+ weight operand prep) -> window GEMMs (paper
Solution A or B by the threshold rule of Alg.2 l.8) -> Solution A's format
fix, i.e. one mec_conv_forward_ex call through the C ABI.

Default workload (N=1): BASELINE.json configs[2], VGG-16 conv1_2
I 64x224x224x64, K 3x3x64x64, stride 1 -- the largest single-GPU config --
in bf16 (the JSON line's `value`), with the same config in tf32 (closest to
the paper's fp32) measured in the same run and reported under "tf32".
Synthetic inputs from the counter-based generator (synth/), generated on the
device.

Multi-GPU (torchrun, one process per GPU; Alg.2 runs every loop "in parallel"
over the images): --scaling strong (default) shards the
configured global batch i_n over the ranks with dist.shard (rank r owns the
global images [r i_n/g, (r+1) i_n/g)); --scaling weak gives every rank a full
batch of its own.  K is broadcast once from rank 0 with NCCL, no other
collective is on the path; time = max over ranks of the device-timed steps.

L2 (126 MB) is flushed before every timed step (a 2x L2 write, then a 2x L2
read so the write's dirty lines are written back outside the step's events).

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
# configs measured a second time in tf32 in the same run (BASELINE.json configs[2]: "bf16 and tf32")
TF32_SIBLING = {"C2": "C2_tf32"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["mec", "reference"], default="mec")
    ap.add_argument("--config", default="C2", help="synth.configs.CONFIGS key (default C2)")
    ap.add_argument("--batch", type=int, default=None, help="override the global batch i_n")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: shard the global batch over the ranks; weak: a full batch per rank")
    ap.add_argument("--path", choices=["auto", "A", "B", "fused", "fastest"], default="auto",
                    help="auto: the paper's Alg.2 l.8 choice (the headline); fastest: MEC_PATH_FASTEST")
    ap.add_argument("--sola-fix", choices=["epilogue", "literal"], default="epilogue")
    ap.add_argument("--T", type=int, default=100)
    ap.add_argument("--rows-per-tile", type=int, default=0,
                    help="window GEMM output rows per tile (multi-row schedule; 0 = library default)")
    ap.add_argument("--gemm-kernel", type=int, default=0,
                    help="window-GEMM kernel: 0 auto, 1 one window per tile, 2 h-sweep, 3 CTA pair")
    ap.add_argument("--split-k", type=int, default=0, help="CTA-pair kernel K ranges (0 = automatic)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tf32", action="store_true", help="skip the tf32 variant of the config")
    ap.add_argument("--no-tf32-peak", action="store_true", help="skip the in-run tf32 peak measurement")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="image chunks of the e2e host-buffer call (copies pipelined with the kernels; "
                         "0 = mec.auto_chunks: ~48 MB of copies per chunk, 4-16)")
    ap.add_argument("--no-flush", action="store_true", help="(diagnostic) do not flush L2")
    ap.add_argument("--no-fused-alt", action="store_true",
                    help="with --path auto, skip measuring the fused path alongside (north_star (3))")
    return ap.parse_args(argv)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def load_ncu(workload_name):
    """Per-kernel ncu metrics of this workload from the committed captures
    (profiles/ncu_metrics.json, written by tools/profile_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_metrics.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get(workload_name, {})


def workload(cfg):
    i_n, i_h, i_w, i_c = cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"]
    k_h, k_w, k_c, s_h, s_w = cfg["k_h"], cfg["k_w"], cfg["k_c"], cfg["s_h"], cfg["s_w"]
    o_h = (i_h - k_h) // s_h + 1
    o_w = (i_w - k_w) // s_w + 1
    flops = 2 * i_n * o_h * o_w * k_h * k_w * i_c * k_c
    return dict(shape=(i_n, i_h, i_w, i_c, k_h, k_w, k_c), o_h=o_h, o_w=o_w, flops=flops,
                nI=i_n * i_h * i_w * i_c, nK=k_h * k_w * i_c * k_c, nO=i_n * o_h * o_w * k_c,
                nL=i_n * o_w * i_h * k_w * i_c, nIm2col=i_n * o_h * o_w * k_h * k_w * i_c)


def rank_work(global_batch: int, rank: int, ws: int, scaling: str) -> dict:
    """The images this rank processes (host logic, tested on CPU with gloo).

    strong: the configured global batch is sharded (dist.shard), rank r owns
    global images [b, e); weak: every rank runs a full batch of its own, at
    global images [r B, (r+1) B).  `index_offset_images` is the global image
    index of the rank's first image (the synthetic generator indexes globally,
    so every shard is a slice of the single-GPU tensor)."""
    from paper_1706_06873_b200 import dist

    if scaling == "strong":
        b, e = dist.shard(global_batch, rank, ws)
        return {"n0": b, "n_local": e - b, "global_batch": global_batch}
    return {"n0": rank * global_batch, "n_local": global_batch, "global_batch": global_batch * ws}


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


def cpu_sample_plan(t1_s: float, cores: int, i_n: int, run_target_s: float = 1.0,
                    budget_s: float = 60.0) -> dict:
    """n_sub images so one threaded run takes >= ~1 s; the mean of
    10 runs (the paper's method) when both timed functions fit the
    budget, else 3 runs.  t1_s = one image on one core."""
    n_img = max(1, min(i_n, 4 * cores, math.ceil(run_target_s * cores / max(t1_s, 1e-4))))
    threads = max(1, min(cores, n_img))
    run_s = t1_s * math.ceil(n_img / threads)
    runs = 10 if 2 * 10 * run_s <= budget_s else 3
    return {"images": n_img, "threads": threads, "runs": runs, "est_run_s": run_s}


def cpu_baseline(cfg, w, dtype_name, seed):
    """The oracle (as it stands) on a bounded sample of the workload: Alg.2
    lowering + Solution-B window GEMMs (oracle.conv_solB), and the direct
    convolution definition (oracle.direct_conv), fp64, threads over images."""
    import oracle
    import synth

    cores = os.cpu_count() or 1
    kind = synth.KIND_GRID8 if dtype_name == "bf16" else synth.KIND_GRID11
    K = synth.kernel_tensor(cfg, kind, seed)
    per_img = w["flops"] / cfg["i_n"]
    I1 = synth.input_images(cfg, 0, 1, kind, seed)
    t0 = time.perf_counter()
    oracle.conv_solB(I1, K, cfg["s_h"], cfg["s_w"], n_threads=1)
    t1 = time.perf_counter() - t0
    plan = cpu_sample_plan(t1, cores, cfg["i_n"])
    n_img, threads, runs = plan["images"], plan["threads"], plan["runs"]
    I = synth.input_images(cfg, 0, n_img, kind, seed)
    out = {}
    for name, fn in (("conv_solB", oracle.conv_solB), ("direct_conv", oracle.direct_conv)):
        ts = []
        for _ in range(runs):
            t0 = time.perf_counter()
            fn(I, K, cfg["s_h"], cfg["s_w"], n_threads=threads)
            ts.append(time.perf_counter() - t0)
        m = statistics.mean(ts)
        out[name] = {"mean_s": m, "runs": runs, "tflops": n_img * per_img / m / 1e12,
                     "s_per_image": m / n_img}
    val = out["conv_solB"]["tflops"]
    return {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{n_img} of {cfg['i_n']} images of {cfg['name']} per run, mean of {runs} runs: "
                      f"oracle.conv_solB (Alg.2 lowering + Solution B window GEMMs, plain C, fp64), "
                      f"{threads} threads; oracle.direct_conv timed the same way",
            "images": n_img, "host_cores_total": cores, "functions": out,
            "extrapolated_full_batch_s": out["conv_solB"]["mean_s"] * cfg["i_n"] / n_img}


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
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
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based generator, seed %d)" % seed,
        "config": {"workload": cfg["name"], "global_batch": cfg["i_n"], "sample_images_per_step": n_img,
                   "same_config": n_img == cfg["i_n"]},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_tf32_peak(dev):
    """tf32 dense peak measured the MEASURED_PEAKS way -- torch.matmul
    fp32 with allow_tf32, 8192^3, best of 10 (a measurement, not on the path)."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def measure(args, cfg, rw, rank, ws, dev, peaks, peak_src, tf32_peak, primary=True):
    """Times the hot path on this rank's images of `cfg`; returns the line fields."""
    import torch

    import synth
    from paper_1706_06873_b200 import dist, mec
    from paper_1706_06873_b200._lib import (MEC_PATH_AUTO, MEC_PATH_FASTEST, MEC_PATH_FUSED, MEC_PATH_SOLUTION_A,
                                            MEC_PATH_SOLUTION_B, MEC_SOLA_FIX_EPILOGUE, MEC_SOLA_FIX_LITERAL,
                                            MecError)

    cfg_local = dict(cfg, i_n=rw["n_local"])
    w = workload(cfg_local)
    w_glob = workload(dict(cfg, i_n=rw["global_batch"]))
    dtype_name = "bf16" if cfg["dtype"] == "bf16" else "tf32"
    tdt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    elt = 2 if dtype_name == "bf16" else 4
    kind = synth.KIND_GRID8 if dtype_name == "bf16" else synth.KIND_GRID11
    seed = synth.SEED_BASE + cfg["index"]
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = w["shape"]
    s_h, s_w = cfg["s_h"], cfg["s_w"]
    path = {"auto": MEC_PATH_AUTO, "A": MEC_PATH_SOLUTION_A, "B": MEC_PATH_SOLUTION_B,
            "fused": MEC_PATH_FUSED, "fastest": MEC_PATH_FASTEST}[args.path]
    fix = MEC_SOLA_FIX_EPILOGUE if args.sola_fix == "epilogue" else MEC_SOLA_FIX_LITERAL
    K_steps = args.steps

    # ---- inputs: this rank's images (global index offset), K from rank 0 by NCCL broadcast
    I = torch.empty((i_n, i_h, i_w, i_c), dtype=tdt, device=dev)
    mec.synth_fill(I, seed, synth.TENSOR_I, kind, index_offset=rw["n0"] * i_h * i_w * i_c)
    K = torch.empty((k_h, k_w, i_c, k_c), dtype=tdt, device=dev)
    if rank == 0:
        mec.synth_fill(K, seed, synth.TENSOR_K, kind)
    dist.broadcast_weights(K, 0)
    K_local = torch.empty_like(K)
    mec.synth_fill(K_local, seed, synth.TENSOR_K, kind)
    k_bcast_ok = bool(torch.equal(K, K_local))
    del K_local
    O = torch.empty((i_n, w["o_h"], w["o_w"], k_c), dtype=tdt, device=dev)
    ws_bytes = mec.workspace_bytes(w["shape"], s_h, s_w, tdt, path=path, T=args.T, sola_fix=fix,
                                   rows_per_tile=args.rows_per_tile, gemm_kernel=args.gemm_kernel,
                                   split_k=args.split_k)
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(4 * l2, 128 << 20), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        return mec.conv_forward(I, K, s_h, s_w, out=O, path=path, T=args.T, sola_fix=fix,
                                rows_per_tile=args.rows_per_tile, workspace=workspace, stage_events=evs,
                                return_path=True, return_gemm=True, gemm_kernel=args.gemm_kernel,
                                split_k=args.split_k)

    # ---- memory: device-memory delta of one pooled call (the library allocates L itself)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    mec.conv_forward(I, K, s_h, s_w, out=O, path=path, T=args.T, sola_fix=fix, rows_per_tile=args.rows_per_tile,
                     gemm_kernel=args.gemm_kernel, split_k=args.split_k)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(dev)[0]
    pooled_delta = max(0, free0 - free1)

    # ---- warm-up
    for _ in range(max(args.warmup, 0)):
        if not args.no_flush:
            mec.l2_flush(flush)
        _, chosen, gemm_kernel = step()
    split_used = mec.conv_forward(I, K, s_h, s_w, out=O, path=path, T=args.T, sola_fix=fix,
                                  rows_per_tile=args.rows_per_tile, workspace=workspace, gemm_kernel=args.gemm_kernel,
                                  split_k=args.split_k, return_split=True)[1]
    torch.cuda.synchronize()
    launches_per_step = mec.last_launch_count()

    # ---- timed region: K steps, CUDA events on the launching stream around each
    # step only (events between the step's kernels would serialise the window
    # GEMM's programmatic dependent launch)
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
    value = w_glob["flops"] * K_steps / (tot_ms * 1e-3) / 1e12

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
    literal = chosen == MEC_PATH_SOLUTION_A and fix == MEC_SOLA_FIX_LITERAL
    fix_ms = [e[2].elapsed_time(e[3]) for e in evs] if literal else None

    # ---- CUDA-graph replay of the same step (launch gaps removed), diagnostic
    graph_ms = None
    if primary:
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
            del g
        except Exception as e:  # noqa: BLE001
            graph_ms = f"unavailable: {e}"

    # ---- end to end through the public API with host buffers (pinned), copies timed:
    # mec_conv_forward_host copies I and K in and O out inside the call, pipelined over
    # image chunks on three streams (the copies of neighbouring chunks overlap the kernels)
    e2e = None
    if primary and not args.no_e2e:
        I_h = I.cpu().pin_memory()
        K_h = K.cpu().pin_memory()
        O_h = torch.empty(O.shape, dtype=O.dtype).pin_memory()
        nch = (max(1, min(args.e2e_chunks, I.shape[0])) if args.e2e_chunks > 0
               else mec.auto_chunks(I.shape[0], (I.numel() + O.numel()) * I.element_size()))
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
        e2e = {"value": w_glob["flops"] * K_steps / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": (w["nI"] + w["nK"]) * elt, "d2h_bytes_per_step": w["nO"] * elt,
               "ms_per_step": e2e_ms / K_steps, "api": "mec_conv_forward_host",
               "chunks": nch, "kernels_per_step": e2e_launches / K_steps}
        del I_h, K_h, O_h, scratch

    # ---- roofline of the dominant kernel (algorithmic bytes / flops per launch)
    mean_lower = statistics.mean(lower_ms)
    mean_gemm = statistics.mean(gemm_ms)
    mean_fix = statistics.mean(fix_ms) if fix_ms else None
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
    kernels = {("weight_prep" if fused else "mec_lower"): (mean_lower, "hbm", bytes_lower / (mean_lower * 1e-3) / 1e9,
                                                          hbm, "GB/s", bytes_lower)}
    t_mem, t_tc = bytes_gemm / (hbm * 1e9), flops / (tc * 1e12)
    gname = "fused_window_gemm" if fused else "window_gemm"
    if t_mem >= t_tc:
        kernels[gname] = (mean_gemm, "hbm", bytes_gemm / (mean_gemm * 1e-3) / 1e9, hbm, "GB/s", bytes_gemm)
    else:
        kernels[gname] = (mean_gemm, "tensor", flops / (mean_gemm * 1e-3) / 1e12, tc, "TFLOP/s", flops)
    if literal:
        bfix = 4 * w["nO"] * elt
        kernels["sola_format_fix"] = (mean_fix, "hbm", bfix / (mean_fix * 1e-3) / 1e9, hbm, "GB/s", bfix)
    dom = max(kernels, key=lambda k: kernels[k][0])
    ms, bound, ach, peak, unit, alg = kernels[dom]
    ncu = load_ncu(cfg["name"])
    nk = ncu.get(dom, {})
    roof = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
            "traffic": nk.get("dram_bytes"), "kernel": dom, "kernel_ms": ms, "algorithmic_per_launch": alg,
            "peak_source": peak_src if bound == "hbm" else f"{tc_src} ({peak_src})",
            "traffic_source": nk.get("source"),
            "all_kernels": {k: {"ms": v[0], "bound": v[1], "achieved": v[2], "unit": v[4],
                                "frac": v[2] / v[3], "algorithmic_per_launch": v[5]} for k, v in kernels.items()}}
    # the same fraction against the nominal B200 figures SURVEY 8(d) asks to
    # report beside the measured ones (north_star: "~8 TB/s"; 2.25 PF/s dense
    # bf16, tf32 half), and against the sustained bf16 measurement
    nom = 8000.0 if bound == "hbm" else (2250.0 if dtype_name == "bf16" else 1125.0)
    roof["nominal"] = {"peak": nom, "unit": unit, "frac": ach / nom,
                       "source": "B200 nominal: HBM 8 TB/s, dense bf16 2.25 PF/s (tf32 x 1/2)"}
    if bound == "tensor" and peaks.get("bf16_tflops_sustained"):
        sus = peaks["bf16_tflops_sustained"] * (1.0 if dtype_name == "bf16" else 0.5)
        roof["frac_of_sustained"] = ach / sus
    g_flops_rate = flops / (mean_gemm * 1e-3) / 1e12
    tpu = {"gemm_tflops": g_flops_rate, "of_dense_peak": g_flops_rate / tc, "peak_tflops": tc,
           "peak_source": f"{tc_src} ({peak_src})",
           "ncu_sm__pipe_tensor_cycles_active_pct": ncu.get(gname, {}).get("tensor_pipe_pct"),
           "ncu_source": ncu.get(gname, {}).get("source")}
    if dtype_name == "tf32" and tf32_peak:
        tpu["of_tf32_peak_measured_in_run"] = g_flops_rate / tf32_peak
        tpu["tf32_peak_measured_in_run_tflops"] = tf32_peak

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
                         "value": w_glob["flops"] * K_steps / (f_tot * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "ms_per_step": f_tot / K_steps,
                         "stages_ms": {"weight_prep": f_prep, "fused_window_gemm": f_gemm},
                         "roofline": f_roof, "gpu_launches": mec.last_launch_count() * K_steps}
        except MecError as e:
            fused_alt = {"path": "fused_lowering_in_gemm", "unavailable": str(e)}

    names = {MEC_PATH_SOLUTION_A: "solution_A_batch_folded", MEC_PATH_SOLUTION_B: "solution_B_per_image",
             MEC_PATH_FUSED: "fused_lowering_in_gemm"}
    stages = {"lower": mean_lower, "gemm": mean_gemm}
    if literal:
        stages["format_fix"] = mean_fix
    res = {
        "value": value, "ms_per_step": tot_ms / K_steps, "dtype": dtype_name,
        "data": f"synthetic (counter-based generator on device, seed {seed}, GRID values exact in {dtype_name})",
        "config": {
            "workload": cfg["name"], "global_batch": rw["global_batch"], "i_n_per_gpu": i_n,
            "first_image": rw["n0"], "I": [i_n, i_h, i_w, i_c], "K": [k_h, k_w, i_c, k_c], "stride": [s_h, s_w],
            "O": [i_n, w["o_h"], w["o_w"], k_c],
            "path": names.get(chosen, str(chosen)),
            "path_rule": f"Alg.2 l.8: Solution A iff o_w <= T={args.T} and #O <= #L" if path == MEC_PATH_AUTO
            else "forced",
            "north_star_letter": "B" if chosen == MEC_PATH_SOLUTION_A else "A",
            "sola_fix": args.sola_fix if chosen == MEC_PATH_SOLUTION_A else None,
            "window_gemm_kernel": {1: "one_window_per_tile", 2: "h_sweep", 3: "cta_pair_split_k"}.get(
                gemm_kernel, str(gemm_kernel)),
            "split_k": split_used if gemm_kernel == 3 else None,
            "l2": "flushed before every timed step: a 2x L2 write, then a 2x L2 read that writes its dirty "
                  "lines back (outside the timed region)" if not args.no_flush else "warm (not flushed)",
            "parallelism": f"dp{ws} ({args.scaling} scaling: images sharded per GPU, K broadcast once by NCCL)",
        },
        "lowered_bytes": {
            "mec_L": w["nL"] * elt, "im2col_L": w["nIm2col"] * elt,
            "im2col_over_mec": w["nIm2col"] / w["nL"], "workspace_allocated": ws_bytes,
            "pooled_call_device_mem_delta": pooled_delta,
        },
        "stages_ms": stages,
        "stages_timing": "per-kernel CUDA events in a separate run of K steps (kernels serialised); "
                         "value / ms_per_step time whole steps with no events inside them",
        "graph_ms_per_step": graph_ms,
        "roofline": roof,
        "tensor_pipe_util": tpu,
        "e2e": e2e,
        "fused_path": fused_alt,
        "gpu_launches": launches_per_step * K_steps,
        "gpu_launches_detail": {"per_step": launches_per_step,
                                "l2_flush_kernels": 0 if args.no_flush else 2 * K_steps},
        "clocks": sampler.summary(),
        "k_broadcast_verified": k_bcast_ok,
    }
    del I, K, O, workspace, flush
    torch.cuda.empty_cache()
    return res


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import synth
    from paper_1706_06873_b200 import dist

    rank, ws, dev = dist.init()
    if dev.type != "cuda":
        raise SystemExit("bench.py needs CUDA GPUs (no CPU fallback)")
    cfg = synth.config(args.config, args.batch)
    rw = rank_work(cfg["i_n"], rank, ws, args.scaling)
    peaks, peak_src = load_peaks()
    want_tf32 = cfg["dtype"] != "bf16" or (args.config in TF32_SIBLING and not args.no_tf32)
    tf32_peak = measure_tf32_peak(dev) if (want_tf32 and not args.no_tf32_peak) else None

    line = {"metric": METRIC, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None}
    res = measure(args, cfg, rw, rank, ws, dev, peaks, peak_src, tf32_peak, primary=True)
    line.update(res)
    if args.config in TF32_SIBLING and not args.no_tf32:
        cfg32 = synth.config(TF32_SIBLING[args.config], args.batch)
        r32 = measure(args, cfg32, rank_work(cfg32["i_n"], rank, ws, args.scaling), rank, ws, dev, peaks,
                      peak_src, tf32_peak, primary=False)
        line["tf32"] = {k: r32[k] for k in ("value", "ms_per_step", "dtype", "config", "stages_ms", "roofline",
                                             "tensor_pipe_util", "fused_path", "lowered_bytes", "clocks",
                                             "gpu_launches")}
        line["gpu_launches"] += r32["gpu_launches"]
    if tf32_peak:
        line["tf32_peak_measured_in_run"] = {"tflops": tf32_peak,
                                             "how": "torch.matmul fp32, allow_tf32, 8192^3, best of 10"}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, workload(cfg), line["dtype"], synth.SEED_BASE + cfg["index"])
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}
    line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
