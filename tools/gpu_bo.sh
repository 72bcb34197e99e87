#!/bin/bash
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 30"
: > gpurun_out/bo.json
for b in 0 100 500 2000; do MEC_EPI_BACKOFF=$b $B >> gpurun_out/bo.json 2>>gpurun_out/bo.err; MEC_EPI_BACKOFF=$b $B --config C3 >> gpurun_out/bo.json 2>>gpurun_out/bo.err; done
for b in 0 500; do echo "== bo $b" >> gpurun_out/bo_trace.txt; MEC_EPI_BACKOFF=$b MEC_DEBUG_FLAGS=197 timeout 300 python tools/trace_gemm.py --config C1 --quiet 2>&1 | grep -E "span|MMA issue" >> gpurun_out/bo_trace.txt; done
