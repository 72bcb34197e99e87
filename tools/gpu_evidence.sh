#!/bin/bash
# Round evidence on one B200 (run under gpurun): GPU parity tests, smoke, the
# default bench line (C2 bf16 + tf32), the reference arm, the C3 / C4 lines,
# the ncu launch list of the default command and full captures of the
# dominant kernels.  Every step under its own timeout.
#   usage: tools/gpu_evidence.sh [tag]      (outputs in gpurun_out/)
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
: > gpurun_out/bench_cfgs.json
for c in C1 C3; do $B --config $c >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err; done
for c in cv1 cv2 cv3 cv4 cv5 cv6 cv7 cv8 cv9 cv10 cv11 cv12 r50_1x1_256to64 r50_1x1_64to256 g_3a_1x1_192to64; do
  $B --config C4_$c --batch 128 --no-fused-alt >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err
done
for c in cv4 cv5 cv12; do $B --config C4_$c --batch 1024 --no-fused-alt --steps 5 >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_gemm|window_gemm|lower_kernel|wide_gemm" -s 6 -c 4 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fused-alt --no-tf32 --no-tf32-peak > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
