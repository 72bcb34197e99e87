"""Summarize bench JSON lines (one per line) into a table."""
import json, sys
for fn in sys.argv[1:]:
    for line in open(fn):
        line=line.strip()
        if not line.startswith("{"): continue
        d=json.loads(line)
        if "impl" in d: print("reference", d["value"]); continue
        r=d["roofline"]; st=d["stages_ms"]; ak=r["all_kernels"]
        fr=" ".join(f"{k}:{v['achieved']:.0f}{v['unit'][:2]}({v['frac']:.2f})" for k,v in ak.items())
        e2e=d.get("e2e") or {}
        print(f"{d['config']['workload']:24s} {d['config']['path'][:10]:10s} {d['dtype']:4s} val={d['value']:7.1f} TF/s ms={d['ms_per_step']*1e3:8.1f}us "
              f"lower={st['lower']*1e3:7.1f} gemm={st['gemm']*1e3:7.1f} fix={st['format_fix']*1e3:6.1f} graph={d['graph_ms_per_step'] if isinstance(d['graph_ms_per_step'],str) else round(d['graph_ms_per_step']*1e3,1)} e2e={e2e.get('value',0):.1f} | {fr}")
