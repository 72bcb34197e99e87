for ch in 2 3 4 6; do timeout 200 python bench.py --config C1 --no-cpu-baseline --no-tf32 --no-tf32-peak --no-fused-alt --steps 20 --e2e-chunks $ch 2>>gpurun_out/c1e2e.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); e=d['e2e']
  print(d['config']['workload'], 'chunks', e.get('chunks'), 'e2e ms', round(e['ms_per_step'],4), 'TF/s', round(e['value'],2), 'step us', round(d['ms_per_step']*1e3,1))
" >> gpurun_out/c1e2e.txt; done
timeout 120 python tools/pcie_probe.py >> gpurun_out/c1e2e.txt 2>&1
