#!/bin/bash
# iteration: parity tests (lowering, multi-row, C1), C1/cv3/cv2 bench, rows-per-tile sweep, lowering trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "lowering or C1 or small_shapes or table2 or stride or multi_row or worked or format_fix" > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
: > gpurun_out/q_bench.json
$B >> gpurun_out/q_bench.json 2>> gpurun_out/q_bench.err
for c in C4_cv3 C4_cv2; do $B --config $c --batch 128 >> gpurun_out/q_bench.json 2>> gpurun_out/q_bench.err; done
for c in C3 C2; do for r in 1 2 4; do $B --config $c --rows-per-tile $r >> gpurun_out/q_bench.json 2>> gpurun_out/q_bench.err; done; done
python tools/trace_lower.py > gpurun_out/trace_lower.txt 2>&1
