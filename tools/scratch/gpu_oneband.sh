#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lower or C1 or cv1 or cv3 or cv7" > gpurun_out/oneband_tests.log 2>&1; echo "rc=$?" >> gpurun_out/oneband_tests.log
MEC_LOWER_ONE_BAND=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lower or C1 or cv1 or cv3 or cv7" >> gpurun_out/oneband_tests.log 2>&1; echo "rc=$?" >> gpurun_out/oneband_tests.log
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/oneband.json
for e in "X=0" "MEC_LOWER_ONE_BAND=1" "MEC_LOWER_ONE_BAND=1 MEC_LOWER_HB=4" "MEC_LOWER_ONE_BAND=1 MEC_LOWER_HB=16" "MEC_LOWER_HB=16"; do
  env $e $B --config C1 >> gpurun_out/oneband.json 2>> gpurun_out/oneband.err
  for c in cv1 cv3 cv7; do env $e $B --config C4_$c --batch 128 >> gpurun_out/oneband.json 2>> gpurun_out/oneband.err; done
done
