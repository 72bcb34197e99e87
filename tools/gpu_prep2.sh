#!/bin/bash
# prep CTAs = max(SMs, tiles/4): check on the layers of the prep sweep, then the GPU tests
mkdir -p gpurun_out
: > gpurun_out/prep2.json
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
for c in "C1" "C3" "C4_cv12 --batch 128" "C4_cv6 --batch 128" "C4_cv5 --batch 128" "C4_cv11 --batch 128" "C4_cv10 --batch 128" "C4_cv9 --batch 128"; do
  $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg': d['config']['workload'], 'us': d['ms_per_step']*1e3, 'lower': d['stages_ms']['lower']*1e3}))" >> gpurun_out/prep2.json 2>> gpurun_out/prep2.err
done
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
