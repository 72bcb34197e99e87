#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "lower or padded or full_batch or table2 or C4_sweep_b128 or stride or small_shapes or sweep_gemm_vs" > gpurun_out/gath_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gath_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
: > gpurun_out/gath_bench.json
if grep -q "rc=0" gpurun_out/gath_tests.log; then
for r in 1 0; do
  MEC_LOWER_GATHER=$r $B --config C1 >> gpurun_out/gath_bench.json 2>> gpurun_out/gath_bench.err
  for c in cv1 cv2 cv3 cv7; do MEC_LOWER_GATHER=$r $B --config C4_$c --batch 128 >> gpurun_out/gath_bench.json 2>> gpurun_out/gath_bench.err; done
done
fi
