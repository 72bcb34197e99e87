B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for H in 0 16 24 32; do for c in "C1" "C4_cv1 --batch 128"; do echo "HB=$H $c" >> gpurun_out/hb.txt; if [ $H = 0 ]; then X=""; else X="MEC_LOWER_HB=$H"; fi; env $X $B --config $c 2>>gpurun_out/hb.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/hb.txt; done; done
