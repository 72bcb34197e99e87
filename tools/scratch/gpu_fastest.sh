#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fastest or fused or abi" > gpurun_out/fastest_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fastest_tests.log
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10 --path fastest"
: > gpurun_out/fastest.json
for c in C1 C2 C3; do $B --config $c >> gpurun_out/fastest.json 2>> gpurun_out/fastest.err; done
for c in cv3 cv8 cv9 cv12; do $B --config C4_$c --batch 128 >> gpurun_out/fastest.json 2>> gpurun_out/fastest.err; done
