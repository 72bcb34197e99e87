#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_sweep or sweep_gemm_vs" > gpurun_out/psaps_tests.log 2>&1; echo "rc=$?" >> gpurun_out/psaps_tests.log
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/psaps_bench.json
if grep -q "rc=0" gpurun_out/psaps_tests.log; then
for a in 1 2 3; do
  MEC_PS_APS=$a $B --config C2_tf32 >> gpurun_out/psaps_bench.json 2>> gpurun_out/psaps_bench.err
  MEC_PS_APS=$a $B --config C4_cv4 --batch 128 >> gpurun_out/psaps_bench.json 2>> gpurun_out/psaps_bench.err
  MEC_PS_APS=$a $B --config C4_cv8 --batch 128 >> gpurun_out/psaps_bench.json 2>> gpurun_out/psaps_bench.err
  MEC_PS_APS=$a $B --config C2 --gemm-kernel 4 >> gpurun_out/psaps_bench.json 2>> gpurun_out/psaps_bench.err
done
fi
