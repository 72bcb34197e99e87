timeout 900 python -m pytest tests -m gpu -x -q -k "pair_sweep or cv4 or C2 or abi" > gpurun_out/pytest_b3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b3.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
for E in 1 0; do for c in "C4_cv4 --batch 128" "C4_cv4 --batch 1024 --steps 3"; do echo "B3=$E $c" >> gpurun_out/b3.txt; MEC_PS_B3=$E $B --config $c 2>>gpurun_out/b3.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'gemm frac', round(d['roofline']['frac'],3))
" >> gpurun_out/b3.txt; done; done
timeout 200 python tools/trace_pair_sweep.py --config C4_cv4 --batch 128 2>&1 | tail -4 >> gpurun_out/b3.txt
