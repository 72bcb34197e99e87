#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair or table2_layers or C4_sweep_b128 or C4_tf32" > gpurun_out/widemn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/widemn_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/widemn_bench.json
if grep -q "rc=0" gpurun_out/widemn_tests.log; then
for c in cv12 cv6 cv11 cv5 cv10; do
  for kt in 0 1; do MEC_WIDE_KT=$kt $B --config C4_$c --batch 128 >> gpurun_out/widemn_bench.json 2>> gpurun_out/widemn_bench.err; done
  for kt in 0 1; do MEC_WIDE_KT=$kt $B --config C4_$c --batch 1024 --steps 5 >> gpurun_out/widemn_bench.json 2>> gpurun_out/widemn_bench.err; done
done
fi
