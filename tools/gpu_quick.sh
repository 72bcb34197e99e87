#!/bin/bash
# quick iteration: parity tests, bench lines (two-kernel and fused), ncu capture of C1 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e"
$B --steps 30 > gpurun_out/q_c1.json 2> gpurun_out/q.err
$B --steps 30 --path fused >> gpurun_out/q_c1.json 2>> gpurun_out/q.err
for c in "C3" "C3 --path fused" "C2 --path fused" "C2_tf32"; do $B --config $c --steps 10 >> gpurun_out/q_c1.json 2>> gpurun_out/q.err; done
for c in C4_cv1 C4_cv2 C4_cv3 C4_cv7; do $B --config $c --batch 128 --steps 10 --path fused >> gpurun_out/q_c1.json 2>> gpurun_out/q.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 4 -c 2 -o gpurun_out/prof_q python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --path fused > gpurun_out/ncu_q.log 2>&1
tail -2 gpurun_out/q.err
