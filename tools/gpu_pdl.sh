#!/bin/bash
# PDL A/B: full GPU tests, then C1 / C3 / cv1 on both paths with and without PDL
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/pdl_tests.txt
: > gpurun_out/pdl.json
for pdl in 0 1; do
  if [ $pdl = 0 ]; then export MEC_NO_PDL=1; else unset MEC_NO_PDL; fi
  for c in "C1" "C1 --path fused" "C3" "C3 --path fused" "C4_cv1 --batch 128 --path fused"; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 --config $c >> gpurun_out/pdl.json 2>/dev/null
  done
done
