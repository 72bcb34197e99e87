#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_sweep" > gpurun_out/ps_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ps_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/ps_bench.json
if grep -q "rc=0" gpurun_out/ps_tests.log; then
for c in C2 C2_tf32 C3; do
  for g in 0 4; do $B --config $c --gemm-kernel $g >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err; done
done
for c in cv8 cv9 cv3; do
  for g in 0 4; do $B --config C4_$c --batch 128 --gemm-kernel $g >> gpurun_out/ps_bench.json 2>> gpurun_out/ps_bench.err; done
done
fi
