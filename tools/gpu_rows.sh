#!/bin/bash
# multi-row window GEMM: R = 1..4 on the configs whose shift allows it
: > gpurun_out/rows.json
for c in "C2" "C3" "C2_tf32" "C4_cv9 --batch 128" "C4_cv8 --batch 128"; do
  for r in 1 2 3 4; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --config $c --rows-per-tile $r >> gpurun_out/rows.json 2>/dev/null
  done
done
