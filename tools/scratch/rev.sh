B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for rep in 1 2; do for E in 1 0; do for c in "C2" "C3" "C4_cv7 --batch 128"; do echo "REV=$E $c" >> gpurun_out/rev.txt; MEC_SWEEP_REV=$E $B --config $c 2>>gpurun_out/rev.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/rev.txt; done; done; done
MEC_SWEEP_REV=1 timeout 600 python -m pytest tests -m gpu -x -q -k "sweep or C2 or C3 or C1 or balanced" > gpurun_out/pytest_rev.log 2>&1; echo rc=$? >> gpurun_out/pytest_rev.log
