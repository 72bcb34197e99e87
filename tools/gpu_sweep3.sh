#!/bin/bash
# sweep GEMM iteration: parity suite, traces, bench lines (every step under its own timeout)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
timeout 60 python tools/trace_sweep.py --config C3 > gpurun_out/tr_c3.txt 2>&1
timeout 60 python tools/trace_sweep.py --config C1 > gpurun_out/tr_c1.txt 2>&1
B="timeout 100 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
: > gpurun_out/s_bench.json
for c in C1 C3 C2 C2_tf32; do $B --config $c >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
for c in C4_cv1 C4_cv3 C4_cv7 C4_cv9 C4_cv10; do $B --config $c --batch 128 >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
