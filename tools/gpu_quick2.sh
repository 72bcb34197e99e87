#!/bin/bash
# quick loop: lowering/conv parity tests, then C1 stage timings and the bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "lowering or C1 or small_shapes or table2 or stride" > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
MEC_LOWER_NO_COPIES=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 --no-fused-alt > gpurun_out/q_bench_old.json 2>> gpurun_out/q_bench.err
for c in C4_cv3 C4_cv2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --no-fused-alt --config $c --batch 128 >> gpurun_out/q_bench.json 2>> gpurun_out/q_bench.err; done
