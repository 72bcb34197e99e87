"""Print the key fields of bench JSON lines (a file of them)."""
import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        c = d["config"]
        print(f"{c['workload']:>22} path={c.get('path','')[:12]:12} rpt={c.get('rows_per_tile', '-')} ms={d['ms_per_step']*1e3:8.1f}us "
              f"TF/s={d['value']:7.1f} stages={ {k: round(v*1e3,1) for k,v in d.get('stages_ms',{}).items()} } "
              f"frac={ {k: round(v['frac'],3) for k,v in d['roofline'].get('all_kernels',{}).items()} }")
