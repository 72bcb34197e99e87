#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/sanitize_cases.py C1 sweep2 tf32 fused > gpurun_out/cg_quick.log 2>&1; echo "rc=$?" >> gpurun_out/cg_quick.log
if grep -q "rc=0" gpurun_out/cg_quick.log; then
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or table2 or full_batch or fused_path or small_shapes or stride" > gpurun_out/cg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cg_tests.log
export MEC_NO_BUILD=1
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
: > gpurun_out/cg_bench.json
cp paper_1706_06873_b200/libmec.so /tmp/libmec_new.so
for v in new base; do
  cp /tmp/libmec_$v.so paper_1706_06873_b200/libmec.so 2>/dev/null || cp paper_1706_06873_b200/libmec_base.so paper_1706_06873_b200/libmec.so
  for c in C1 C2 C3; do $B --config $c >> gpurun_out/cg_bench.json 2>> gpurun_out/cg_bench.err; done
  for c in cv1 cv3 cv7 cv9; do $B --config C4_$c --batch 128 --no-fused-alt >> gpurun_out/cg_bench.json 2>> gpurun_out/cg_bench.err; done
done
fi
