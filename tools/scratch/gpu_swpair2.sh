#!/bin/bash
mkdir -p gpurun_out
cp paper_1706_06873_b200/libmec_plainwait.so paper_1706_06873_b200/libmec.so
export MEC_NO_BUILD=1
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/swpair_bench2.json
timeout 120 env MEC_SWEEP_PAIR=1 python tools/sanitize_cases.py C1 sweep2 > gpurun_out/swpair_quick2.log 2>&1
for c in C1 C2 C3; do MEC_SWEEP_PAIR=1 $B --config $c >> gpurun_out/swpair_bench2.json 2>> gpurun_out/swpair_bench2.err; done
for c in C1 C2 C3; do MEC_SWEEP_PAIR=1 MEC_SWEEP_ISSUERS=1 $B --config $c >> gpurun_out/swpair_bench2.json 2>> gpurun_out/swpair_bench2.err; done
