#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/s4.txt
for b in 0 50 200 1000; do
  echo "== backoff $b" >> gpurun_out/s4.txt
  MEC_SWEEP_BACKOFF=$b timeout 60 python tools/trace_sweep.py --config C3 2>&1 | tail -4 >> gpurun_out/s4.txt
done
echo "== nomma" >> gpurun_out/s4.txt
MEC_SWEEP_DBG=2 timeout 60 python tools/trace_sweep.py --config C3 2>&1 | tail -4 >> gpurun_out/s4.txt
echo "== nomma, no copier st" >> gpurun_out/s4.txt
MEC_SWEEP_DBG=6 timeout 60 python tools/trace_sweep.py --config C3 2>&1 | tail -4 >> gpurun_out/s4.txt
echo "== no epilogue stores" >> gpurun_out/s4.txt
MEC_SWEEP_DBG=1 timeout 60 python tools/trace_sweep.py --config C3 2>&1 | tail -4 >> gpurun_out/s4.txt
