"""Regenerate DESIGN.md section 12's results and ncu tables from the committed
evidence (profiles/r2_bench_default.json, profiles/r2_bench_cfgs.json,
profiles/ncu_metrics.json), so the document quotes exactly what profiles/ holds.
usage: python tools/design_tables.py"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, *a)
R1 = {"C2": "611", "C1": "31.7", "C3": "168", "cv4_b128": "2185", "cv5_b128": "82.5", "cv6_b128": "51.2",
      "cv8_b128": "501", "cv9_b128": "91.4", "cv12_b128": "48.2", "cv4_b1024": "18123"}
KER = {"h_sweep": "h-sweep", "4": "pair sweep", "cta_pair_split_k": "CTA pair", "one_window_per_tile": "one window"}
ONE = {"r50_1x1_256to64": "1×1 56²·256→64", "r50_1x1_64to256": "1×1 56²·64→256", "g_3a_1x1_192to64": "1×1 28²·192→64"}


def frac(ak):
    g = ak["window_gemm"]
    return f"{g['frac']:.2f} {'HBM' if g['bound'] == 'hbm' else 'TC'}"


def results():
    d = json.loads(open(P("profiles", "r2_bench_default.json")).read().strip().splitlines()[-1])
    rows = [json.loads(l) for l in open(P("profiles", "r2_bench_cfgs.json"))]
    out = ["| config | path / GEMM kernel | step µs (r1) | TF/s | GEMM frac | lowering frac | fused µs |",
           "|---|---|---|---|---|---|---|"]
    ak = d["roofline"]["all_kernels"]
    f = d["fused_path"]
    out.append(f"| **C2 VGG conv1_2 b64 (headline)** | B / h-sweep | **{d['ms_per_step'] * 1e3:.0f}** (611) | "
               f"**{d['value']:.0f}** | {frac(ak)} | **{ak['mec_lower']['frac']:.2f}** | "
               f"{f['ms_per_step'] * 1e3:.0f} ({f['value']:.0f} TF/s) |")
    t = d["tf32"]
    akt = t["roofline"]["all_kernels"]
    tf = t.get("fused_path", {}).get("ms_per_step")
    out.append(f"| **C2 tf32** | B / pair sweep | **{t['ms_per_step'] * 1e3:.0f}** (1934) | **{t['value']:.0f}** | "
               f"{frac(akt)} | **{akt['mec_lower']['frac']:.2f}** | {tf * 1e3:.0f} |" if tf else "—")
    names = {"C1_alexnet_conv1": ("C1 AlexNet conv1 b32", "C1"), "C3_resnet50_stage2_3x3": ("C3 ResNet-50 3×3 b256", "C3")}
    for r in rows:
        w = r["config"]["workload"]
        a = r["roofline"]["all_kernels"]
        if w in names:
            lab, key = names[w]
        else:
            m = re.match(r"C4_(.*)_b(\d+)", w)
            lay, b = m.group(1), m.group(2)
            lab, key = ONE.get(lay, lay) + f" b{b}", f"{lay}_b{b}"
        pl = "A" if "solution_A" in r["config"]["path"] else "B"
        fz = r.get("fused_path") or {}
        fz = f"{fz['ms_per_step'] * 1e3:.0f}" if fz.get("ms_per_step") else "—"
        old = f" ({R1[key]})" if key in R1 else ""
        out.append(f"| {lab} | {pl} / {KER.get(r['config']['window_gemm_kernel'], r['config']['window_gemm_kernel'])} | "
                   f"{r['ms_per_step'] * 1e3:.1f}{old} | {r['value']:.0f} | {frac(a)} | {a['mec_lower']['frac']:.2f} | {fz} |")
    return "\n".join(out)


def ncu():
    d = json.load(open(P("profiles", "ncu_metrics.json")))
    order = [("C2_vgg16_conv1_2", "C2"), ("C2_vgg16_conv1_2_tf32", "C2 tf32"), ("C1_alexnet_conv1", "C1"),
             ("C3_resnet50_stage2_3x3", "C3"), ("C4_cv5_b128", "cv5 b128"), ("C4_cv6_b128", "cv6 b128"),
             ("C4_cv11_b128", "cv11 b128"), ("C4_cv12_b128", "cv12 b128"), ("C4_cv8_b128", "cv8 b128")]

    def kn(n):
        for k, v in (("lower_rows_kernel", "row copy"), ("lower_kernel", "staged"), ("sweep_gemm", "h-sweep"),
                     ("pair_sweep", "pair sweep"), ("wide_gemm", "CTA pair")):
            if k in n:
                return v
        return n[:20]
    out = ["| workload | kernel | µs | DRAM read / write MB | L2→SM (TMA) MB | tensor pipe |", "|---|---|---|---|---|---|"]
    for key, lab in order:
        for st in ("mec_lower", "window_gemm"):
            m = d.get(key, {}).get(st)
            if not m:
                continue
            name = f"lowering ({kn(m['kernel_name'])})" if st == "mec_lower" else kn(m["kernel_name"])
            tma = f"{m['l2_to_sm_tma_bytes'] / 1e6:.0f}" if m["l2_to_sm_tma_bytes"] else "—"
            tp = f"{m['tensor_pipe_pct']:.0f}%" if m["tensor_pipe_pct"] else "—"
            out.append(f"| {lab} | {name} | {m['duration_us']:.1f} | {m['dram_read'] / 1e6:.0f} / {m['dram_write'] / 1e6:.0f} "
                       f"| {tma} | {tp} |")
    return "\n".join(out)


def readme_table():
    d = json.loads(open(P("profiles", "r2_bench_default.json")).read().strip().splitlines()[-1])
    rows = {json.loads(l)["config"]["workload"]: json.loads(l) for l in open(P("profiles", "r2_bench_cfgs.json"))}
    ak = lambda x: x["roofline"]["all_kernels"]
    t, c1, c3 = d["tf32"], rows["C1_alexnet_conv1"], rows["C3_resnet50_stage2_3x3"]
    cv4, cv4k = rows["C4_cv4_b128"], rows["C4_cv4_b1024"]
    b = [rows[f"C4_{l}_b1024"] for l in ("cv5", "cv6", "cv11", "cv12")]
    g = lambda x: f"{ak(x)['window_gemm']['frac']:.2f}"
    steps = " / ".join(f"{x['ms_per_step'] * 1e3:.0f}" for x in b)
    tfs = " / ".join(f"{x['value']:.0f}" for x in b)
    gemms = " / ".join(g(x) for x in b)
    return "\n".join([
        "| workload | step | TF/s | dominant kernel vs roofline |",
        "|---|---|---|---|",
        f"| VGG-16 conv1_2 b64, bf16 (headline) | {d['ms_per_step'] * 1e3:.0f} µs | {d['value']:.0f} | window GEMM {g(d)}, "
        f"lowering {ak(d)['mec_lower']['frac']:.2f} of measured HBM; fused path {d['fused_path']['ms_per_step'] * 1e3:.0f} µs "
        f"({d['fused_path']['value']:.0f} TF/s) |",
        f"| VGG-16 conv1_2 b64, tf32 | {t['ms_per_step']:.2f} ms | {t['value']:.0f} | GEMM {g(t)} (round 1: 0.38), lowering "
        f"{ak(t)['mec_lower']['frac']:.2f} of HBM |",
        f"| AlexNet conv1 b32 | {c1['ms_per_step'] * 1e3:.1f} µs | {c1['value']:.0f} | GEMM {g(c1)} of HBM (latency-bound small step) |",
        f"| ResNet-50 3×3 b256 | {c3['ms_per_step'] * 1e3:.0f} µs | {c3['value']:.0f} | GEMM {g(c3)} of HBM; fused "
        f"{c3['fused_path']['ms_per_step'] * 1e3:.0f} µs |",
        f"| cv4 (7×7 s2) b128 / b1024 | {cv4['ms_per_step'] * 1e3:.0f} µs / {cv4k['ms_per_step']:.1f} ms | {cv4['value']:.0f} / "
        f"{cv4k['value']:.0f} | GEMM {g(cv4)} / {g(cv4k)} of HBM |",
        f"| cv5 / cv6 / cv11 / cv12 at b1024 | {steps} µs | {tfs} | GEMM {gemms} of the bf16 peak |",
    ]), d


def replace_table(s, header, new):
    a = s.index(header)
    b = s.index("\n\n", a)
    return s[:a] + new + s[b:]


def main():
    path = P("DESIGN.md")
    s = open(path).read()
    s = replace_table(s, "| config | path / GEMM kernel | step µs (r1) |", results())
    s = replace_table(s, "| workload | kernel | µs | DRAM read / write MB |", ncu())
    open(path, "w").write(s)
    tbl, d = readme_table()
    rp = P("README.md")
    r = open(rp).read()
    r = replace_table(r, "| workload | step | TF/s | dominant kernel vs roofline |", tbl)
    r = re.sub(r"VGG conv1_2 b64 at [0-9.]+ ms \([0-9.]+ TF/s;",
               f"VGG conv1_2 b64 at {d['e2e']['ms_per_step']:.1f} ms ({d['e2e']['value']:.1f} TF/s;", r)
    open(rp, "w").write(r)
    print(results())


if __name__ == "__main__":
    main()
