timeout 900 python -m pytest tests -m gpu -x -q -k "pair_sweep or cv4 or C2 or fused or fastest or balanced" > gpurun_out/pytest_prod.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_prod.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 10"
for c in "C2" "C2_tf32" "C3" "C4_cv4 --batch 128 --no-fused-alt" "C4_cv8 --batch 128" "C4_cv9 --batch 128"; do echo "$c" >> gpurun_out/prod.txt; $B --config $c 2>>gpurun_out/prod.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); f=d.get('fused_path') or {}
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'gemm frac', round(d['roofline']['frac'],3), 'fused', round(f.get('ms_per_step',0)*1e3,1))
" >> gpurun_out/prod.txt; done
