#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 10 --warmup 3"
: > gpurun_out/s2.json
for c in C1 C3; do
  for d in 0 1 2 4 7 3 5 6; do echo "{\"dbg\": $d}" >> gpurun_out/s2.json; MEC_SWEEP_DBG=$d $B --config $c >> gpurun_out/s2.json 2>> gpurun_out/s2.err; done
  for h in 2 4 8 16; do echo "{\"H\": $h}" >> gpurun_out/s2.json; MEC_SWEEP_H=$h $B --config $c >> gpurun_out/s2.json 2>> gpurun_out/s2.err; done
done
