B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
for A in 1 2 3; do for c in "C4_cv4 --batch 128" "C4_cv8 --batch 128" "C2_tf32"; do echo "APS=$A $c" >> gpurun_out/aps.txt; MEC_PS_APS=$A $B --config $c 2>>gpurun_out/aps.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'gemm frac', round(d['roofline']['frac'],3))
" >> gpurun_out/aps.txt; done; done
