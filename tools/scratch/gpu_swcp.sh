#!/bin/bash
mkdir -p gpurun_out
export MEC_SWEEP_CP=1
timeout 120 python tools/sanitize_cases.py C1 sweep2 tf32 fused > gpurun_out/swcp_quick.log 2>&1; echo "rc=$?" >> gpurun_out/swcp_quick.log
if grep -q "rc=0" gpurun_out/swcp_quick.log; then
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or table2 or full_batch or fused_path or small_shapes or stride" > gpurun_out/swcp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/swcp_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
: > gpurun_out/swcp_bench.json
for cp in 1 0; do
  for c in C1 C2 C3; do MEC_SWEEP_CP=$cp $B --config $c >> gpurun_out/swcp_bench.json 2>> gpurun_out/swcp_bench.err; done
  for c in cv1 cv3 cv7 cv9; do MEC_SWEEP_CP=$cp $B --config C4_$c --batch 128 --no-fused-alt >> gpurun_out/swcp_bench.json 2>> gpurun_out/swcp_bench.err; done
done
fi
