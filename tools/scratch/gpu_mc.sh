#!/bin/bash
mkdir -p gpurun_out
export MEC_WIDE_MC=2
timeout 120 python tools/sanitize_cases.py wide > gpurun_out/mc_quick.log 2>&1; echo "rc=$?" >> gpurun_out/mc_quick.log
if grep -q "rc=0" gpurun_out/mc_quick.log; then
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_pair or C4_sweep_b128" > gpurun_out/mc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mc_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/mc_bench.json
for mc in 2 1; do
  for c in cv12 cv6 cv11 cv5 cv10; do MEC_WIDE_MC=$mc $B --config C4_$c --batch 128 >> gpurun_out/mc_bench.json 2>> gpurun_out/mc_bench.err; done
  for c in cv5 cv12; do MEC_WIDE_MC=$mc $B --config C4_$c --batch 1024 --steps 5 >> gpurun_out/mc_bench.json 2>> gpurun_out/mc_bench.err; done
done
fi
