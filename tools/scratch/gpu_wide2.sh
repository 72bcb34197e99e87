#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair or table2_layers or C4_sweep_b128 or b1024" > gpurun_out/wide_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/wide_bench.json
for c in cv12 cv6 cv11 cv5 cv10; do
  $B --config C4_$c --batch 128 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
  $B --config C4_$c --batch 128 --gemm-kernel 3 --split-k 2 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
  $B --config C4_$c --batch 1024 --steps 5 >> gpurun_out/wide_bench.json 2>> gpurun_out/wide_bench.err
done
