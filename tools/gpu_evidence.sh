#!/bin/bash
# Round evidence: GPU parity tests, the default bench line, the reference arm,
# the ncu launch list of the same command and one full capture of the
# dominant kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"window_gemm|lower_kernel" -s 6 -c 3 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fused-alt > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
