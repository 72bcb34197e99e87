"""Summarise ncu captures into profiles/ (committed evidence).

usage:
  python tools/profile_summary.py --launches gpurun_out/launches_c1.csv \
      --full gpurun_out/prof_c1.ncu-rep --config C1_alexnet_conv1 --tag r1 [--steps 3]

Writes profiles/<tag>_<config>_launches.csv (per-launch device times, cold
cache, serialised), profiles/<tag>_<config>_ncu.txt (key metrics per kernel
of the --set full capture) and merges per-launch DRAM traffic
(dram__bytes_read.sum + dram__bytes_write.sum) into profiles/traffic.json,
which bench.py reports as roofline.traffic.
"""
import argparse
import csv
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
]


def short(name):
    for k in ("lower_rows_kernel", "lower_rows_gather_kernel", "lower_kernel", "window_gemm_kernel", "sweep_gemm_kernel", "wide_gemm_kernel", "pair_sweep_kernel",
              "copy16_kernel", "block_permute_kernel", "flush_kernel", "synth_kernel", "fused"):
        if k in name:
            # every window-GEMM kernel is the "window_gemm" stage of bench.py
            return {"lower_kernel": "mec_lower", "lower_rows_kernel": "mec_lower", "lower_rows_gather_kernel": "mec_lower",
                    "window_gemm_kernel": "window_gemm",
                    "sweep_gemm_kernel": "window_gemm", "wide_gemm_kernel": "window_gemm",
                    "pair_sweep_kernel": "window_gemm",
                    "copy16_kernel": "sola_copy", "block_permute_kernel": "sola_transpose"}.get(k, k)
    return name[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--config", required=True)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--fused", action="store_true",
                    help="the capture ran MEC_PATH_FUSED: name kernels as bench.py does (weight_prep, "
                         "fused_window_gemm) and suffix the output files with _fused")
    args = ap.parse_args()
    if args.fused:
        global short
        plain = short

        def short(name):  # noqa: F811
            k = plain(name)
            return {"mec_lower": "weight_prep", "window_gemm": "fused_window_gemm"}.get(k, k)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    base = os.path.join(ROOT, "profiles", f"{args.tag}_{args.config}" + ("_fused" if args.fused else ""))
    if args.launches:
        rows = [r for r in csv.reader(open(args.launches)) if r]
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        out = [["id", "kernel", "duration_ns"]]
        per = defaultdict(list)
        for r in rows[hdr + 1:]:
            if len(r) != len(h):
                continue
            d = dict(zip(h, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "ns")
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "nsecond": 1, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
            out.append([d["ID"], short(d["Kernel Name"]), f"{ns:.0f}"])
            per[short(d["Kernel Name"])].append(ns)
        with open(base + "_launches.csv", "w") as f:
            csv.writer(f).writerows(out)
        with open(base + "_launches_summary.txt", "w") as f:
            step_kernels = ("mec_lower", "window_gemm", "sola_copy", "sola_transpose", "weight_prep",
                            "fused_window_gemm")
            tot = sum(sum(v) for k, v in per.items() if k in step_kernels)
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, {args.config}\n")
            f.write("# cold-cache serialised launches: compare shares, not absolutes\n")
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                share = (sum(v) / tot) if k in step_kernels and tot else 0
                f.write(f"{k:16s} launches={len(v):3d} mean_us={sum(v) / len(v) / 1e3:8.2f} share_of_step={share:.2f}\n")
    if args.full:
        raw = subprocess.run(["ncu", "-i", args.full, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, units = rows[0], rows[1]
        traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
        traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        lines = [f"# ncu --set full --clock-control none, {args.config} ({args.full})"]
        acc = defaultdict(list)
        for r in rows[2:]:
            name = short(r[h.index("Kernel Name")])
            lines.append(f"== {name}")
            for k in KEYS:
                if k in h:
                    lines.append(f"   {k} = {r[h.index(k)]} {units[h.index(k)]}")
            def val(k):
                v = float(r[h.index(k)].replace(",", ""))
                u = units[h.index(k)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            def num(k):
                try:
                    return float(r[h.index(k)].replace(",", ""))
                except (ValueError, IndexError):
                    return None
            acc[name].append({
                "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                "dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
                "tensor_pipe_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                "l2_to_sm_tma_bytes": val("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum")
                if "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum" in h else None,
                "duration_us": val("gpu__time_duration.sum") / 1e3 if units[h.index("gpu__time_duration.sum")] == "ns"
                else val("gpu__time_duration.sum"),
                "kernel_name": r[h.index("Kernel Name")][:120],
            })
        with open(base + "_ncu.txt", "w") as f:
            f.write("\n".join(lines) + "\n")
        traffic.setdefault(args.config, {})
        metrics_path = os.path.join(ROOT, "profiles", "ncu_metrics.json")
        metrics = json.load(open(metrics_path)) if os.path.exists(metrics_path) else {}
        metrics.setdefault(args.config, {})
        for k, v in acc.items():
            traffic[args.config][k] = sum(x["dram_bytes"] for x in v) / len(v)
            m = {key: (sum(x[key] for x in v) / len(v) if all(isinstance(x[key], float) for x in v) else v[-1][key])
                 for key in v[-1]}
            m["launches_averaged"] = len(v)
            m["source"] = os.path.relpath(base + "_ncu.txt", ROOT)
            metrics[args.config][k] = m
        with open(traffic_path, "w") as f:
            json.dump(traffic, f, indent=1, sort_keys=True)
        with open(metrics_path, "w") as f:
            json.dump(metrics, f, indent=1, sort_keys=True)
    print("wrote", base + "*")


if __name__ == "__main__":
    main()
