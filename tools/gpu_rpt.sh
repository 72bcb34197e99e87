#!/bin/bash
# multi-row tile sweep (rows_per_tile) on the stride-1 configs
mkdir -p gpurun_out
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
: > gpurun_out/rpt.json
for c in C3 C2 C4_cv9 C4_cv8; do
  for r in 1 2 4 8; do
    echo "== $c R=$r" >> gpurun_out/rpt.json
    $B --config $c --rows-per-tile $r $( [ $c = C4_cv9 -o $c = C4_cv8 ] && echo --batch 128 ) 2>>gpurun_out/rpt.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])" >> gpurun_out/rpt.json
  done
done
