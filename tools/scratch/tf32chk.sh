B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32-peak --no-fused-alt --steps 20 --config C2_tf32"
for rep in 1 2; do for E in auto 0; do echo "PSBAL=$E rep $rep" >> gpurun_out/tf32chk.txt; if [ $E = auto ]; then X=""; else X="MEC_PS_BALANCED=0"; fi; env $X $B 2>>gpurun_out/tf32chk.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'gemm frac', round(d['roofline']['frac'],3))
" >> gpurun_out/tf32chk.txt; done; done
for m in resnet101 stride; do timeout 600 python tools/workloads.py $m --steps 5 --out profiles/r2_next_$m.json > gpurun_out/next_$m.log 2>&1; done
mkdir -p gpurun_out/profiles_next; cp profiles/r2_next_*.json gpurun_out/profiles_next/ 2>/dev/null
