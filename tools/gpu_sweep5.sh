#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
B="timeout 100 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20"
: > gpurun_out/s_bench.json
for i in 1 2; do
for c in C1 C3 C2; do MEC_SWEEP_ISSUERS=$i $B --config $c >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
for c in C4_cv1 C4_cv3 C4_cv7 C4_cv9; do MEC_SWEEP_ISSUERS=$i $B --config $c --batch 128 >> gpurun_out/s_bench.json 2>> gpurun_out/s_bench.err; done
done
