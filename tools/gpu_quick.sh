#!/bin/bash
# quick iteration: parity tests, C1/C3 bench lines, ncu capture of C1 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/q_c1.json 2> gpurun_out/q.err
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 20 --no-e2e >> gpurun_out/q_c1.json 2>> gpurun_out/q.err
timeout 300 python bench.py --config C4_cv7 --batch 128 --no-cpu-baseline --steps 10 --no-e2e >> gpurun_out/q_c1.json 2>> gpurun_out/q.err
timeout 300 python bench.py --config C4_cv12 --batch 128 --no-cpu-baseline --steps 10 --no-e2e >> gpurun_out/q_c1.json 2>> gpurun_out/q.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 4 -c 2 -o gpurun_out/prof_q python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_q.log 2>&1
tail -2 gpurun_out/q.err
