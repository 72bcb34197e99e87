#!/bin/bash
# One gpurun session for the round's evidence: the default bench line, every
# config on the paper path and the fused path, the cv-layer sweep, ncu launch
# lists and full captures (C1 two-kernel and fused).
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.csv
timeout 400 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20"
: > gpurun_out/bench_paths.json
for c in C1 C2 C2_tf32 C3; do
  for p in auto fused; do $B --config $c --path $p >> gpurun_out/bench_paths.json 2>> gpurun_out/bench_more.err; done
done
$B --config C1 --path B >> gpurun_out/bench_paths.json 2>> gpurun_out/bench_more.err
$B --config C3 --path B >> gpurun_out/bench_paths.json 2>> gpurun_out/bench_more.err
: > gpurun_out/bench_sweep128.json
for c in C4_cv1 C4_cv2 C4_cv3 C4_cv4 C4_cv5 C4_cv6 C4_cv7 C4_cv8 C4_cv9 C4_cv10 C4_cv11 C4_cv12; do
  for p in auto fused; do
    timeout 300 python bench.py --config $c --batch 128 --path $p --no-cpu-baseline --no-e2e --steps 10 >> gpurun_out/bench_sweep128.json 2>> gpurun_out/bench_more.err
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1_fused.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --path fused > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 4 -c 2 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 4 -c 2 -o gpurun_out/prof_c1_fused python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --path fused > gpurun_out/ncu_full_fused.log 2>&1
ls -la gpurun_out
