#!/bin/bash
for r in 1 2 4; do MEC_DEBUG_R=$r MEC_DEBUG_FLAGS=0 timeout 300 python tools/trace_gemm.py --quiet --config C3 --batch 64 | grep -E "span|FLAGS|epilogue us"; done
