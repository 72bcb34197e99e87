#!/bin/bash
# Copy one tools/gpu_evidence.sh run (gpurun_out/) into profiles/ under a tag:
# bench lines, ncu launch lists and full-capture summaries, sanitizer logs.
# usage: tools/evidence_collect.sh [tag]   (default r2)
T=${1:-r2}
cd "$(dirname "$0")/.."
cp gpurun_out/bench_default.json profiles/${T}_bench_default.json
cp gpurun_out/bench_ref.json profiles/${T}_bench_ref.json
cp gpurun_out/bench_cfgs.json profiles/${T}_bench_cfgs.json
for t in memcheck racecheck synccheck; do [ -f gpurun_out/sanitize_$t.log ] && ! grep -q "is closed on this pool" gpurun_out/sanitize_$t.log && cp gpurun_out/sanitize_$t.log profiles/${T}_sanitize_$t.log; done
python tools/profile_summary.py --launches gpurun_out/launches_c2.csv --config C2_vgg16_conv1_2 --tag $T
python tools/profile_summary.py --launches gpurun_out/launches_c2_tf32.csv --config C2_vgg16_conv1_2_tf32 --tag $T
declare -A NAME=([C2]=C2_vgg16_conv1_2 [C2_tf32]=C2_vgg16_conv1_2_tf32 [C1]=C1_alexnet_conv1
                 [C3]=C3_resnet50_stage2_3x3 [C4_cv5]=C4_cv5_b128 [C4_cv6]=C4_cv6_b128 [C4_cv11]=C4_cv11_b128
                 [C4_cv12]=C4_cv12_b128 [C4_cv8]=C4_cv8_b128)
for c in "${!NAME[@]}"; do
  [ -f gpurun_out/prof_$c.ncu-rep ] && python tools/profile_summary.py --full gpurun_out/prof_$c.ncu-rep --config ${NAME[$c]} --tag $T
done
