#!/bin/bash
mkdir -p gpurun_out
export MEC_NO_BUILD=1
B="timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-tf32 --no-tf32-peak --no-fused-alt --steps 10"
: > gpurun_out/psreg.json
cp paper_1706_06873_b200/libmec.so /tmp/libmec_cur.so
for v in cur old cur old; do
  if [ $v = old ]; then cp paper_1706_06873_b200/libmec_old_ps.so paper_1706_06873_b200/libmec.so; else cp /tmp/libmec_cur.so paper_1706_06873_b200/libmec.so; fi
  MEC_PS_APS=1 $B --config C2_tf32 >> gpurun_out/psreg.json 2>> gpurun_out/psreg.err
  MEC_PS_APS=1 $B --config C4_cv4 --batch 128 >> gpurun_out/psreg.json 2>> gpurun_out/psreg.err
done
