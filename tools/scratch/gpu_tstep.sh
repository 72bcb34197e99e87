#!/bin/bash
mkdir -p gpurun_out
for c in C1 C3; do timeout 300 python tools/trace_step.py --config $c > gpurun_out/tstep_$c.log 2>&1; done
timeout 300 python tools/trace_step.py --config C4_cv1 --batch 128 > gpurun_out/tstep_cv1.log 2>&1
