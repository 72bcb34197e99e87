#!/bin/bash
# Round evidence on one B200 (run under gpurun): GPU parity tests, smoke, the
# default bench line (C2 bf16 + tf32), the reference arm, the C1 / C3 / C4
# lines, the ncu launch list of the default command, full ncu captures of the
# dominant kernels per config, and compute-sanitizer runs.  Every step under
# its own timeout.   usage: tools/gpu_evidence.sh [parts]   (default: all)
# (compute-sanitizer is closed on this pool since round 2: sanitize only on request)
PARTS=${1:-"tests bench cfgs ncu"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi.csv
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
fi
if has bench; then
  timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
if has cfgs; then
  B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 20"
  : > gpurun_out/bench_cfgs.json
  for c in C1 C3; do $B --config $c >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err; done
  for c in cv1 cv2 cv3 cv4 cv5 cv6 cv7 cv8 cv9 cv10 cv11 cv12 r50_1x1_256to64 r50_1x1_64to256 g_3a_1x1_192to64; do
    $B --config C4_$c --batch 128 --no-fused-alt >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err
  done
  for c in cv4 cv5 cv6 cv11 cv12; do $B --config C4_$c --batch 1024 --no-fused-alt --steps 5 >> gpurun_out/bench_cfgs.json 2>> gpurun_out/bench_cfgs.err; done
fi
if has ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_tf32.csv python bench.py --config C2_tf32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32-peak --no-fused-alt > /dev/null 2>&1
  K='regex:lower_kernel|lower_rows|sweep_gemm|window_gemm|wide_gemm|pair_sweep'
  NB="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fused-alt --no-tf32 --no-tf32-peak"
  for spec in "C2:" "C2_tf32:" "C1:" "C3:" "C4_cv5:--batch 128" "C4_cv6:--batch 128" "C4_cv11:--batch 128" "C4_cv12:--batch 128" "C4_cv8:--batch 128"; do
    c=${spec%%:*}; extra=${spec#*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k "$K" -s 6 -c 2 -o gpurun_out/prof_$c $NB --config $c $extra > gpurun_out/ncu_$c.log 2>&1
  done
fi
if has sanitize; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  done
fi
ls -la gpurun_out
