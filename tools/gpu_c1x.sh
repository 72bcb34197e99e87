#!/bin/bash
# C1 experiments: box alignment 32 vs 128 bytes, strip padding
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 30"
: > gpurun_out/c1x.json
for i in 1 2; do
$B >> gpurun_out/c1x.json 2>>gpurun_out/c1x.err
MEC_BOX_ALIGN=128 $B >> gpurun_out/c1x.json 2>>gpurun_out/c1x.err
MEC_BOX_ALIGN=64 $B >> gpurun_out/c1x.json 2>>gpurun_out/c1x.err
done
MEC_BOX_ALIGN=128 timeout 300 python -m pytest tests -m gpu -x -q -k "C1 or table2 or small_shapes" > gpurun_out/c1x_tests.log 2>&1
