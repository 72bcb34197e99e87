#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/ps_bench.json
for ch in 0 6 9 12 16 24 37 56; do
  if [ $ch = 0 ]; then E=""; else E="MEC_PS_CHUNKS=$ch"; fi
  env $E $B --config C2_tf32 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
  env $E $B --config C4_cv4 --batch 128 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
  env $E $B --config C2 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
done
