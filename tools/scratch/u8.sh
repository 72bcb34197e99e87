export MEC_NO_BUILD=1
B="timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 20"
run() { for c in "C2" "C3" "C4_cv12 --batch 128" "C4_cv6 --batch 128" "C4_cv11 --batch 128" "C4_cv5 --batch 128" "C4_cv8 --batch 128"; do echo "$1 $c" >> gpurun_out/u8.txt; $B --config $c 2>>gpurun_out/u8.err | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l)
  print(d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'stages', {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})
" >> gpurun_out/u8.txt; done; }
run U4
cp paper_1706_06873_b200/libmec.so /tmp/libmec_u4.so; cp build/u8/libmec.so paper_1706_06873_b200/libmec.so
run U8
cp /tmp/libmec_u4.so paper_1706_06873_b200/libmec.so
