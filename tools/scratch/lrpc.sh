B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for R in 0 2 4; do for c in cv12 cv6 cv11 cv5; do echo "RPC=$R $c" >> gpurun_out/lrpc.txt; if [ $R = 0 ]; then E=""; else E="MEC_LOWER_ROWS_PER_CTA=$R"; fi; env $E $B --config C4_$c --batch 128 2>>gpurun_out/lrpc.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/lrpc.txt; done; done
for P in 1 2 4; do for c in cv12 cv6; do echo "PREP_PER_SM=$P $c" >> gpurun_out/lrpc.txt; MEC_PREP_PER_SM=$P $B --config C4_$c --batch 128 2>>gpurun_out/lrpc.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/lrpc.txt; done; done
