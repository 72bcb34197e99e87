#!/bin/bash
# one gpurun session: bench lines + ncu launch list + ncu full capture (C1)
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.csv
timeout 300 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for c in "C3 --path A" "C3 --path B" "C2" "C2_tf32" "C1 --sola-fix literal" "C1 --path B"; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 >> gpurun_out/bench_more.json 2>> gpurun_out/bench_more.err
done
for c in C4_cv5 C4_cv6 C4_cv11 C4_cv12 C4_cv4 C4_cv8 C4_cv9 C4_cv1 C4_cv3 C4_cv7; do
  timeout 300 python bench.py --config $c --batch 128 --no-cpu-baseline --no-e2e --steps 10 >> gpurun_out/bench_sweep128.json 2>> gpurun_out/bench_more.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 4 -c 2 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
