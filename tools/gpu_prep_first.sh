#!/bin/bash
# prep CTAs first vs last (MEC_PREP_FIRST) now that the prep uses 64 x 64 vector tiles
mkdir -p gpurun_out
: > gpurun_out/prepfirst.json
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
for f in 0 1; do
  for c in "C3" "C4_cv5 --batch 128" "C4_cv9 --batch 128" "C4_cv10 --batch 128" "C4_cv11 --batch 128" "C4_cv3 --batch 128" "C4_cv1 --batch 128"; do
    MEC_PREP_FIRST=$f $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'first': $f, 'cfg': d['config']['workload'], 'us': d['ms_per_step']*1e3, 'lower': d['stages_ms']['lower']*1e3}))" >> gpurun_out/prepfirst.json 2>> gpurun_out/prepfirst.err
  done
done
