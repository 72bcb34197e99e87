#!/bin/bash
# gather-path iteration: its parity tests, a trace, and C1 bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather" 2>&1 | tail -3
MEC_DEBUG_FLAGS=0 timeout 300 python tools/trace_gemm.py --path fused --quiet > gpurun_out/trace_gather.txt 2>&1
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e"
$B --steps 30 > gpurun_out/g_c1.json 2> gpurun_out/g.err
$B --steps 30 --path fused >> gpurun_out/g_c1.json 2>> gpurun_out/g.err
for c in C4_cv1 C4_cv2 C4_cv3 C4_cv7; do $B --config $c --batch 128 --steps 10 --path fused >> gpurun_out/g_c1.json 2>> gpurun_out/g.err; done
tail -2 gpurun_out/g.err
