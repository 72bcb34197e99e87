B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
for E in 1 0; do for c in "C1" "C4_cv1 --batch 128" "C4_cv2 --batch 128" "C4_cv3 --batch 128"; do echo "SPAD=$E $c" >> gpurun_out/spad.txt; if [ $E = 1 ]; then X="MEC_STRIP_PAD=1"; else X=""; fi; env $X $B --config $c 2>>gpurun_out/spad.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], d['config']['window_gemm_kernel'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, d['lowered_bytes']['workspace_allocated'])
" >> gpurun_out/spad.txt; done; done
MEC_STRIP_PAD=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_spad.log 2>&1; echo rc=$? >> gpurun_out/pytest_spad.log
