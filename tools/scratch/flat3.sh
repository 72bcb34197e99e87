timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for E in 1 0; do for c in "C4_r50_1x1_256to64 --batch 128" "C4_g_3a_1x1_192to64 --batch 128"; do echo "FLAT64=$E $c" >> gpurun_out/flat3.txt; MEC_SWEEP_FLAT64=$E $B --config $c 2>>gpurun_out/flat3.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/flat3.txt; done; done
