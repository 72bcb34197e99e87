#!/bin/bash
# sweep GEMM: parity suite, then C1/C2/C3 lines (sweep default vs MEC_SWEEP=0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
: > gpurun_out/s_bench.json
for c in C1 C3 C2 C2_tf32; do $B --config $c >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
for c in C4_cv1 C4_cv3 C4_cv7 C4_cv9 C4_cv10; do $B --config $c --batch 128 >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
for c in C1 C3; do MEC_SWEEP=0 $B --config $c >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
