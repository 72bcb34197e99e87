#!/bin/bash
for f in 0 1 2 4 3 5 7; do MEC_DEBUG_FLAGS=$f timeout 300 python tools/trace_gemm.py --quiet $@; done
