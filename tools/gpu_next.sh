#!/bin/bash
# section 8(f) NEXT rows: stride-sweep parity tests + the three measurement modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stride_sweep" 2>&1 | tail -3 > gpurun_out/next_tests.txt
timeout 900 python tools/workloads.py resnet101 > gpurun_out/next_resnet101.jsonl 2> gpurun_out/next.err
timeout 900 python tools/workloads.py stride > gpurun_out/next_stride.jsonl 2>> gpurun_out/next.err
timeout 1500 python tools/workloads.py paths > gpurun_out/next_paths.jsonl 2>> gpurun_out/next.err
