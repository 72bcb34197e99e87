#!/bin/bash
mkdir -p gpurun_out
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/cv4ab.json
for r in 1 2; do
  (cd build/old && $B --config C4_cv4 --batch 128) >> gpurun_out/cv4ab.json 2>> gpurun_out/cv4ab.err
  $B --config C4_cv4 --batch 128 >> gpurun_out/cv4ab.json 2>> gpurun_out/cv4ab.err
  (cd build/old && $B --config C4_cv8 --batch 128) >> gpurun_out/cv4ab.json 2>> gpurun_out/cv4ab.err
  $B --config C4_cv8 --batch 128 >> gpurun_out/cv4ab.json 2>> gpurun_out/cv4ab.err
done
