#!/bin/bash
mkdir -p gpurun_out
B="timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --steps 10"
: > gpurun_out/fusedcmp.json
for c in C1 C2 C3; do $B --config $c >> gpurun_out/fusedcmp.json 2>> gpurun_out/fusedcmp.err; done
for c in cv1 cv2 cv3 cv4 cv5 cv6 cv7 cv8 cv9 cv10 cv11 cv12; do $B --config C4_$c --batch 128 >> gpurun_out/fusedcmp.json 2>> gpurun_out/fusedcmp.err; done
for c in cv4 cv8 cv9; do $B --config C4_$c --batch 1024 --steps 3 >> gpurun_out/fusedcmp.json 2>> gpurun_out/fusedcmp.err; done
timeout 150 python bench.py --no-cpu-baseline --no-e2e --no-tf32-peak --steps 5 --config C2_tf32 >> gpurun_out/fusedcmp.json 2>> gpurun_out/fusedcmp.err
