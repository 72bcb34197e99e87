#!/bin/bash
# lowering iteration: parity tests, C1/cv3/cv2 bench, C1 lowering ncu capture
mkdir -p gpurun_out
bash tools/gpu_quick2.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lower_kernel -s 3 -c 1 -o gpurun_out/prof_lower_it python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fused-alt > gpurun_out/ncu_lower.log 2>&1
python tools/trace_lower.py > gpurun_out/trace_lower.txt 2>&1
