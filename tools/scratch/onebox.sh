timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
for c in "C1" "C3" "C4_cv1 --batch 128" "C4_cv2 --batch 128" "C4_cv9 --batch 128"; do echo "$c" >> gpurun_out/onebox.txt; $B --config $c 2>>gpurun_out/onebox.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); f=d.get('fused_path') or {}
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'fused', round(f.get('ms_per_step',0)*1e3,1))
" >> gpurun_out/onebox.txt; done
