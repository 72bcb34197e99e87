#!/bin/bash
mkdir -p gpurun_out
K='regex:lower_kernel|lower_rows|sweep_gemm|window_gemm|wide_gemm|pair_sweep'
NB="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fused-alt --no-tf32 --no-tf32-peak"
for c in cv4 cv7; do
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 6 -c 2 -o gpurun_out/prof_C4_$c $NB --config C4_$c --batch 128 > gpurun_out/ncu_C4_$c.log 2>&1
done
