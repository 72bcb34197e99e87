#!/bin/bash
# rows per lowering band x weight-prep CTAs per SM on the small-image, large-K layers
mkdir -p gpurun_out
: > gpurun_out/hbprep.json
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-fused-alt --steps 20 --batch 128"
for c in C4_cv12 C4_cv6 C4_cv5 C4_cv11; do
  for hb in 0 1 2 4 8; do
    for k in 1 4; do
      if [ $hb = 0 ]; then unset MEC_LOWER_HB; else export MEC_LOWER_HB=$hb; fi
      MEC_PREP_PER_SM=$k $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'hb': $hb, 'k': $k, 'cfg': d['config']['workload'], 'us': d['ms_per_step']*1e3, 'lower': d['stages_ms']['lower']*1e3}))" >> gpurun_out/hbprep.json 2>> gpurun_out/hbprep.err
    done
  done
done
