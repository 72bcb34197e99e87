#!/bin/bash
for st in 1 2 3 4; do MEC_DEBUG_STAGES=$st MEC_DEBUG_FLAGS=3 timeout 300 python tools/trace_gemm.py --quiet $@ | grep -E "span|FLAGS"; done
for st in 1 2 4; do MEC_DEBUG_STAGES=$st MEC_DEBUG_FLAGS=0 timeout 300 python tools/trace_gemm.py --quiet $@ | grep -E "span|FLAGS"; done
