#!/bin/bash
# gather-path trace: spinning vs blocking handshakes
for sp in 0 1; do
  MEC_GATHER_SPIN=$sp MEC_DEBUG_FLAGS=0 timeout 300 python tools/trace_gemm.py --path fused --quiet > gpurun_out/gtrace_spin$sp.txt 2>&1
  MEC_GATHER_SPIN=$sp MEC_DEBUG_FLAGS=26 timeout 300 python tools/trace_gemm.py --path fused --quiet > gpurun_out/gtrace_spin${sp}_f26.txt 2>&1
  MEC_GATHER_SPIN=$sp timeout 300 python bench.py --no-cpu-baseline --no-e2e --path fused --steps 30 > gpurun_out/gspin$sp.json 2>/dev/null
done
