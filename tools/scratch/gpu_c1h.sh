#!/bin/bash
mkdir -p gpurun_out
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/c1h.json
for h in 0 2 3 4 6 8 11; do
  if [ $h = 0 ]; then E=""; else E="MEC_SWEEP_H=$h"; fi
  env $E $B --config C1 >> gpurun_out/c1h.json 2>> gpurun_out/c1h.err
done
for i in 1 2; do MEC_SWEEP_ISSUERS=$i $B --config C1 >> gpurun_out/c1h.json 2>> gpurun_out/c1h.err; done
