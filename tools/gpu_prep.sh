#!/bin/bash
# weight-prep CTAs first + prep CTAs per SM sweep
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/prep.json
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
for k in 2 4 8; do
  for c in "C1" "C3" "C4_cv12 --batch 128" "C4_cv6 --batch 128" "C4_cv9 --batch 128" "C4_cv5 --batch 128" "C4_cv8 --batch 128"; do
    MEC_PREP_PER_SM=$k $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'k': $k, 'cfg': d['config']['workload'], 'us': d['ms_per_step']*1e3, 'stages': d['stages_ms']}))" >> gpurun_out/prep.json 2>> gpurun_out/prep.err
  done
done
