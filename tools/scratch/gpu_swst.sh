#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/swst.json
for st in 4 5 6 7 8; do MEC_SWEEP_STAGES=$st $B --config C2 >> gpurun_out/swst.json 2>> gpurun_out/swst.err; done
for st in 6 8; do MEC_SWEEP_EPI_BYTES=64 MEC_SWEEP_STAGES=$st $B --config C2 >> gpurun_out/swst.json 2>> gpurun_out/swst.err; done
for st in 5 8; do MEC_SWEEP_EPI_BYTES=64 MEC_SWEEP_STAGES=$st $B --config C3 >> gpurun_out/swst.json 2>> gpurun_out/swst.err; done
