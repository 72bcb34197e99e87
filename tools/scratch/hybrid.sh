timeout 600 python -m pytest tests -m gpu -x -q -k "hybrid or wide_pair or C4_sweep_b128" > gpurun_out/pytest_hyb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hyb.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for E in 1 0; do for c in cv6 cv11 cv12; do echo "HYB=$E $c" >> gpurun_out/hyb.txt; MEC_WIDE_HYBRID=$E $B --config C4_$c --batch 128 2>>gpurun_out/hyb.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'split', d['config'].get('split_k'), 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/hyb.txt; done; done
