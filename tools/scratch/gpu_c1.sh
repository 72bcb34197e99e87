#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair" > gpurun_out/c1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c1_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/c1_bench.json
if grep -q "rc=0" gpurun_out/c1_tests.log; then
  for g in 0 3; do $B --config C1 --gemm-kernel $g >> gpurun_out/c1_bench.json 2>> gpurun_out/c1_bench.err; done
  for g in 0 3; do $B --config C3 --gemm-kernel $g >> gpurun_out/c1_bench.json 2>> gpurun_out/c1_bench.err; done
  for g in 0 3; do $B --config C4_cv1 --batch 128 --gemm-kernel $g >> gpurun_out/c1_bench.json 2>> gpurun_out/c1_bench.err; done
  for g in 0 3; do $B --config C4_cv9 --batch 128 --gemm-kernel $g >> gpurun_out/c1_bench.json 2>> gpurun_out/c1_bench.err; done
fi
