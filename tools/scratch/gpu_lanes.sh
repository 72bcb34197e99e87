#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or wide or pair or C1 or C2 or C3 or table2" > gpurun_out/lanes_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lanes_tests.log
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/lanes.json
for l in 1 2; do
  MEC_PROD_LANES=$l $B --config C2 >> gpurun_out/lanes.json 2>> gpurun_out/lanes.err
  for c in C1 C3; do MEC_PROD_LANES=$l $B --no-tf32 --config $c >> gpurun_out/lanes.json 2>> gpurun_out/lanes.err; done
  for c in cv12 cv6 cv5 cv11 cv8 cv4; do MEC_PROD_LANES=$l $B --no-tf32 --config C4_$c --batch 128 >> gpurun_out/lanes.json 2>> gpurun_out/lanes.err; done
  for c in cv12 cv5; do MEC_PROD_LANES=$l $B --no-tf32 --config C4_$c --batch 1024 --steps 5 >> gpurun_out/lanes.json 2>> gpurun_out/lanes.err; done
done
