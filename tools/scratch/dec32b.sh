timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for c in cv5 cv6 cv10 cv11 cv12 r50_1x1_256to64 r50_1x1_64to256 g_3a_1x1_192to64; do echo "$c" >> gpurun_out/dec32b.txt; $B --config C4_$c --batch 128 2>>gpurun_out/dec32b.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'gemm frac', round(d['roofline']['frac'],3))
" >> gpurun_out/dec32b.txt; done
