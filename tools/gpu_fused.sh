#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
B="timeout 100 python bench.py --no-cpu-baseline --no-e2e --steps 20"
: > gpurun_out/f_bench.json
for c in C1 C2 C3; do $B --config $c >> gpurun_out/f_bench.json 2>> gpurun_out/f_bench.err; done
for c in C4_cv4 C4_cv8 C4_cv9 C4_cv10; do $B --config $c --batch 128 >> gpurun_out/f_bench.json 2>> gpurun_out/f_bench.err; done
