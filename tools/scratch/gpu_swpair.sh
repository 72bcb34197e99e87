#!/bin/bash
mkdir -p gpurun_out
export MEC_SWEEP_PAIR=1
timeout 300 python tools/sanitize_cases.py C1 sweep2 tf32 fused > gpurun_out/swpair_quick.log 2>&1; echo "rc=$?" >> gpurun_out/swpair_quick.log
if grep -q "rc=0" gpurun_out/swpair_quick.log; then
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or table2 or full_batch or fused_path or small_shapes or stride" > gpurun_out/swpair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/swpair_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
: > gpurun_out/swpair_bench.json
for sp in 0 1; do
  for c in C1 C2 C3; do MEC_SWEEP_PAIR=$sp $B --config $c >> gpurun_out/swpair_bench.json 2>> gpurun_out/swpair_bench.err; done
  for c in cv1 cv3 cv7 cv9; do MEC_SWEEP_PAIR=$sp $B --config C4_$c --batch 128 --no-fused-alt >> gpurun_out/swpair_bench.json 2>> gpurun_out/swpair_bench.err; done
done
fi
