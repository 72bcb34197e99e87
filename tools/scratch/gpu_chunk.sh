#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/chunk_bench.json
for b in 1 2 3 4 6 8 16; do $B --config C2 --batch $b >> gpurun_out/chunk_bench.json 2>> gpurun_out/chunk_bench.err; done
