#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/ps_bench.json
for ef in 0 1; do
  MEC_PS_EVICT_FIRST=$ef $B --config C2_tf32 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
  MEC_PS_EVICT_FIRST=$ef $B --config C4_cv4 --batch 128 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
  MEC_PS_EVICT_FIRST=$ef $B --config C4_cv8 --batch 128 --gemm-kernel 4 >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err
done
