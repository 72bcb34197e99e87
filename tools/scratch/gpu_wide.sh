#!/bin/bash
# CTA-pair kernel: parity first (under a short timeout), then b128 / b1024 timings vs the one-window kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair or table2_layers" > gpurun_out/wide_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests.log
if grep -q "rc=0" gpurun_out/wide_tests.log; then
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/wide_bench.json
for c in cv12 cv6 cv11 cv5 cv10; do
  $B --config C4_$c --batch 128 --gemm-kernel 3 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
  for sk in 1 2 3 4 6; do $B --config C4_$c --batch 128 --gemm-kernel 3 --split-k $sk >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err; done
  MEC_WIDE_NSUB=1 $B --config C4_$c --batch 128 --gemm-kernel 3 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
  $B --config C4_$c --batch 1024 --gemm-kernel 3 --steps 5 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
  MEC_WIDE_NSUB=1 $B --config C4_$c --batch 1024 --gemm-kernel 3 --steps 5 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
done
fi
