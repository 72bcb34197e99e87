#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_sweep or C2 or fastest" > gpurun_out/ps5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ps5_tests.log
rm -f gpurun_out/trace_ps.log
for c in C4_cv8; do timeout 300 python tools/trace_pair_sweep.py --config $c --batch 128 >> gpurun_out/trace_ps.log 2>&1; done
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/ps5.json
$B --config C2 >> gpurun_out/ps5.json 2>> gpurun_out/ps5.err
for c in cv4 cv8; do $B --no-tf32 --config C4_$c --batch 128 >> gpurun_out/ps5.json 2>> gpurun_out/ps5.err; done
$B --no-tf32 --config C4_cv4 --batch 1024 --steps 3 >> gpurun_out/ps5.json 2>> gpurun_out/ps5.err
MEC_PS_BOX3=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_sweep" > gpurun_out/ps5_box3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ps5_box3_tests.log
