#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "lower or padded or full_batch or table2 or C4_sweep_b128" > gpurun_out/rows_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rows_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/rows_bench.json
if grep -q "rc=0" gpurun_out/rows_tests.log; then
for r in 1 0; do
  for c in C2 C2_tf32 C3; do MEC_LOWER_ROWS=$r $B --config $c >> gpurun_out/rows_bench.json 2>> gpurun_out/rows_bench.err; done
  for c in cv4 cv5 cv6 cv8 cv9 cv10 cv11 cv12; do MEC_LOWER_ROWS=$r $B --config C4_$c --batch 128 >> gpurun_out/rows_bench.json 2>> gpurun_out/rows_bench.err; done
done
fi
