#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/swdbg.json
for d in 0 1 2 4 6 7; do MEC_SWEEP_DBG=$d $B --config C2 >> gpurun_out/swdbg.json 2>> gpurun_out/swdbg.err; done
for d in 0 2 6; do MEC_SWEEP_DBG=$d $B --config C3 >> gpurun_out/swdbg.json 2>> gpurun_out/swdbg.err; done
