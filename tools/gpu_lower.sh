#!/bin/bash
# lowering: parity + C1/C4-cv1 timing for several w-loop splits
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lowering or padded_lowering or small_shapes" 2>&1 | tail -2 > gpurun_out/lower_tests.txt
: > gpurun_out/lower_ws.json
for ws in 1 2 3 4 6; do
  MEC_LOWER_WSPLIT=$ws timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 >> gpurun_out/lower_ws.json 2>/dev/null
  MEC_LOWER_WSPLIT=$ws timeout 300 python bench.py --config C4_cv1 --batch 128 --no-cpu-baseline --no-e2e --steps 10 >> gpurun_out/lower_ws.json 2>/dev/null
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 >> gpurun_out/lower_ws.json 2>/dev/null
