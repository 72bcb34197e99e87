#!/bin/bash
# HEAD check: full GPU parity suite, smoke, default bench line, main configs.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
timeout 400 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20"
: > gpurun_out/h_cfgs.json
for c in C2 C2_tf32 C3; do $B --config $c >> gpurun_out/h_cfgs.json 2>> gpurun_out/h_cfgs.err; done
for c in C4_cv5 C4_cv6 C4_cv8 C4_cv12; do $B --config $c --batch 128 >> gpurun_out/h_cfgs.json 2>> gpurun_out/h_cfgs.err; done
