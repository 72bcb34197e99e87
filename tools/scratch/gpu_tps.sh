#!/bin/bash
mkdir -p gpurun_out
for c in C4_cv4 C4_cv8 C2_tf32; do timeout 300 python tools/trace_pair_sweep.py --config $c --batch 128 >> gpurun_out/trace_ps.log 2>&1; done
