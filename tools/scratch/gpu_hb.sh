#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/hb_bench.json
for hb in 0 2 3 4 6; do
  if [ $hb = 0 ]; then E=""; else E="MEC_LOWER_HB=$hb"; fi
  env $E $B --config C2 >> gpurun_out/hb_bench.json 2>> gpurun_out/hb_bench.err
  env $E $B --config C2_tf32 >> gpurun_out/hb_bench.json 2>> gpurun_out/hb_bench.err
  env $E $B --config C3 >> gpurun_out/hb_bench.json 2>> gpurun_out/hb_bench.err
done
