#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair" > gpurun_out/wsplit_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wsplit_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/wsplit.json
if grep -q "rc=0" gpurun_out/wsplit_tests.log; then
for c in cv12 cv6 cv11 cv5 cv10; do
  for s in 1 2 3 4; do
    $B --config C4_$c --batch 128 --split-k $s >> gpurun_out/wsplit.json 2>> gpurun_out/wsplit.err
  done
done
for c in cv12 cv6; do
  for s in 1 2; do
    $B --config C4_$c --batch 1024 --split-k $s --steps 5 >> gpurun_out/wsplit.json 2>> gpurun_out/wsplit.err
  done
done
fi
