#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/trace_sweep.py --config C1 > gpurun_out/trace_c1_sweep.log 2>&1
SW_CYCLES=1 timeout 300 python tools/trace_sweep.py --config C1 >> gpurun_out/trace_c1_sweep.log 2>&1
timeout 300 python tools/trace_lower.py --config C1 > gpurun_out/trace_c1_lower.log 2>&1
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/c1p.json
$B --config C1 >> gpurun_out/c1p.json 2>> gpurun_out/c1p.err
MEC_SWEEP_PAIR=1 $B --config C1 >> gpurun_out/c1p.json 2>> gpurun_out/c1p.err
MEC_LOWER_CTAS_PER_SM=2 $B --config C1 >> gpurun_out/c1p.json 2>> gpurun_out/c1p.err
MEC_LOWER_HB=16 $B --config C1 >> gpurun_out/c1p.json 2>> gpurun_out/c1p.err
MEC_LOWER_HB=4 $B --config C1 >> gpurun_out/c1p.json 2>> gpurun_out/c1p.err
