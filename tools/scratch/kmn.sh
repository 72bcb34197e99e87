B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for E in 1 0; do for c in "C4_cv12 --batch 128" "C4_cv6 --batch 128" "C4_cv11 --batch 128" "C4_cv5 --batch 128" "C4_cv12 --batch 1024 --steps 5" "C4_cv6 --batch 1024 --steps 5"; do echo "KMN=$E $c" >> gpurun_out/kmn.txt; MEC_WIDE_KMN=$E $B --config $c 2>>gpurun_out/kmn.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/kmn.txt; done; done
