"""B200-native hot path of MEC (Cho & Brand, ICML 2017, arXiv 1706.06873).

libmec.so (csrc/, C ABI in include/mec.h) holds every kernel: compact
lowering, tcgen05/TMEM/TMA window GEMMs (Solutions A and B), Solution A's
format fix.  This package is the thin ctypes binding (mec.py) and the
multi-GPU driver (dist.py).
"""
from .mec import (conv_forward, conv_forward_host, host_scratch_bytes, im2col_elems, l2_flush, last_launch_count, lower,  # noqa: F401
                  lowered_elems, out_dims, select_path, synth_fill, workspace_bytes)
from ._lib import MecError  # noqa: F401
