#!/bin/bash
# gather path: accumulator count (A stages = TMEM left / 32, max 8)
for k in 4 3 2; do
  MEC_GATHER_NACC=$k timeout 300 python tools/trace_gemm.py --path fused --quiet > gpurun_out/gtrace_na$k.txt 2>&1
  MEC_GATHER_NACC=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e --path fused --steps 30 > gpurun_out/gna$k.json 2>/dev/null
  MEC_GATHER_NACC=$k timeout 300 python bench.py --config C4_cv1 --batch 128 --no-cpu-baseline --no-e2e --path fused --steps 10 >> gpurun_out/gna$k.json 2>/dev/null
done
