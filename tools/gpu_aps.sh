#!/bin/bash
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 30"
: > gpurun_out/aps.json
for a in 2 1 3 4 6; do echo "aps $a" >> gpurun_out/aps.json; MEC_APS=$a $B >> gpurun_out/aps.json 2>>gpurun_out/aps.err; MEC_APS=$a $B --config C3 >> gpurun_out/aps.json 2>>gpurun_out/aps.err; done
for a in 2 4; do echo "== aps $a" >> gpurun_out/aps_trace.txt; MEC_APS=$a MEC_DEBUG_FLAGS=197 timeout 300 python tools/trace_gemm.py --config C1 --quiet 2>&1 | grep -E "span|MMA issue" >> gpurun_out/aps_trace.txt; done
