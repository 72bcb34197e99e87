#!/bin/bash
# rows_per_tile sweep of the one-window kernel on the layers the h-sweep kernel does not take
mkdir -p gpurun_out
: > gpurun_out/rpt_sweep.json
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
for c in C4_cv4 C4_cv10 C4_cv12 C4_cv6; do
  for r in 0 1 2 3 4 6 8; do
    $B --config $c --batch 128 --rows-per-tile $r >> gpurun_out/rpt_sweep.json 2>> gpurun_out/rpt_sweep.err
  done
done
for r in 0 1 2 4; do $B --config C2_tf32 --rows-per-tile $r >> gpurun_out/rpt_sweep.json 2>> gpurun_out/rpt_sweep.err; done
