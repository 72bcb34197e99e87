#!/bin/bash
mkdir -p gpurun_out
B="timeout 300 python bench.py --no-cpu-baseline --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/e2e.json
for ch in 1 2 4 8 16; do $B --e2e-chunks $ch >> gpurun_out/e2e.json 2>> gpurun_out/e2e.err; done
for ch in 1 2 4 8; do $B --config C1 --e2e-chunks $ch >> gpurun_out/e2e.json 2>> gpurun_out/e2e.err; done
python tools/pcie_probe.py > gpurun_out/pcie.json 2> gpurun_out/pcie.err
