#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/am.json
for am in 0 1; do
  for d in 0 7; do
    if [ $am = 1 ]; then E="MEC_SWEEP_AM=1"; else E="MEC_SWEEP_AMX=0"; fi
    env $E MEC_SWEEP_DBG=$d $B --config C2 >> gpurun_out/am.json 2>> gpurun_out/am.err
  done
done
