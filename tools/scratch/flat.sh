B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for E in 32 129; do for c in "C3" "C1" "C4_cv1 --batch 128" "C4_cv9 --batch 128"; do echo "FLAT_OW=$E $c" >> gpurun_out/flat.txt; MEC_SWEEP_FLAT_OW=$E $B --config $c 2>>gpurun_out/flat.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/flat.txt; done; done
MEC_SWEEP_FLAT_OW=129 timeout 600 python -m pytest tests -m gpu -x -q -k "sweep or C3 or C1 or cv9 or cv1 or balanced or small_shapes or table2" > gpurun_out/pytest_flat.log 2>&1; echo rc=$? >> gpurun_out/pytest_flat.log
