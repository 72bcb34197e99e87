"""ctypes declarations for libmec.so (include/mec.h, include/mec_synth.h).

Loading fails loudly if the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libmec.so")

# mec_status_t
MEC_OK = 0
MEC_ERR_INVALID_ARG = 1
MEC_ERR_UNSUPPORTED = 2
MEC_ERR_MISALIGNED = 3
MEC_ERR_CUDA = 4
MEC_ERR_NO_MEMORY = 5
# mec_dtype_t
MEC_DTYPE_BF16 = 0
MEC_DTYPE_TF32 = 1
# mec_path_t
MEC_PATH_AUTO = 0
MEC_PATH_SOLUTION_A = 1
MEC_PATH_SOLUTION_B = 2
MEC_PATH_FUSED = 3
MEC_PATH_FASTEST = 4  # fused h-sweep where measured faster, else MEC_PATH_AUTO (include/mec.h)
# mec_sola_fix_t
MEC_SOLA_FIX_EPILOGUE = 0
MEC_SOLA_FIX_LITERAL = 1
MEC_SOLA_FIX_NONE = 2
MEC_DEFAULT_T = 100
# mec_synth_kind_t
MEC_SYNTH_GRID8 = 0
MEC_SYNTH_GRID11 = 1
MEC_SYNTH_FULL24 = 2

# Every symbol the headers declare (checked by tests/test_abi_host.py).
EXPORTED = (
    "mec_options_init", "mec_out_dims", "mec_select_path", "mec_lowered_elems",
    "mec_im2col_elems", "mec_workspace_bytes", "mec_lower", "mec_conv_forward",
    "mec_conv_forward_ex", "mec_last_launch_count", "mec_status_string",
    "mec_last_error_message", "mec_abi_version", "mec_synth_fill", "mec_l2_flush",
    "mec_workspace_bytes_ex", "mec_lower_padded", "mec_maxpool", "mec_lower_pitched",
    "mec_host_scratch_bytes", "mec_conv_forward_host",
)
# mec_layout_t
MEC_LAYOUT_NHWC = 0
MEC_LAYOUT_HNWC = 1


class MecShape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("i_n", "i_h", "i_w", "i_c", "k_h", "k_w", "k_c")]


class MecOptions(ctypes.Structure):
    _fields_ = [
        ("path", ctypes.c_int),
        ("T", ctypes.c_int),
        ("sola_fix", ctypes.c_int),
        ("rows_per_tile", ctypes.c_int),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("stage_events", ctypes.c_void_p * 4),
        ("selected_path", ctypes.c_int),
        ("pad_h", ctypes.c_int),
        ("pad_w", ctypes.c_int),
        ("selected_gemm", ctypes.c_int),
        ("gemm_kernel", ctypes.c_int),
        ("split_k", ctypes.c_int),
        ("selected_split", ctypes.c_int),
    ]


_lock = threading.Lock()
_lib = None


def lib():
    """Load libmec.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if os.environ.get("MEC_NO_BUILD") != "1":
            from . import _build

            if not _build.up_to_date():
                _build.build()
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"libmec.so not found at {SO_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH)
        P = ctypes.POINTER
        sp = P(MecShape)
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        L.mec_options_init.argtypes = [P(MecOptions)]
        L.mec_options_init.restype = None
        L.mec_out_dims.argtypes = [sp, ci, ci, P(i64), P(i64)]
        L.mec_out_dims.restype = ci
        L.mec_select_path.argtypes = [sp, ci, ci, ci]
        L.mec_select_path.restype = ci
        L.mec_lowered_elems.argtypes = [sp, ci, ci]
        L.mec_lowered_elems.restype = i64
        L.mec_im2col_elems.argtypes = [sp, ci, ci]
        L.mec_im2col_elems.restype = i64
        L.mec_workspace_bytes.argtypes = [sp, ci, ci, ci]
        L.mec_workspace_bytes.restype = ctypes.c_size_t
        L.mec_lower.argtypes = [vp, vp, sp, ci, ci, ci, vp]
        L.mec_lower.restype = ci
        L.mec_lower_padded.argtypes = [vp, vp, sp, ci, ci, ci, ci, ci, vp]
        L.mec_lower_padded.restype = ci
        L.mec_lower_pitched.argtypes = [vp, vp, sp, ci, ci, i64, ci, vp]
        L.mec_lower_pitched.restype = ci
        L.mec_workspace_bytes_ex.argtypes = [sp, ci, ci, ci, P(MecOptions)]
        L.mec_workspace_bytes_ex.restype = ctypes.c_size_t
        L.mec_maxpool.argtypes = [vp, vp, i64, i64, i64, i64, ci, ci, ci, ci, ci, ci, vp]
        L.mec_maxpool.restype = ci
        L.mec_conv_forward.argtypes = [vp, vp, vp, sp, ci, ci, ci, vp]
        L.mec_conv_forward.restype = ci
        L.mec_conv_forward_ex.argtypes = [vp, vp, vp, sp, ci, ci, ci, vp, P(MecOptions)]
        L.mec_conv_forward_ex.restype = ci
        L.mec_host_scratch_bytes.argtypes = [sp, ci, ci, ci, P(MecOptions), ci]
        L.mec_host_scratch_bytes.restype = ctypes.c_size_t
        L.mec_conv_forward_host.argtypes = [vp, vp, vp, sp, ci, ci, ci, vp, P(MecOptions), ci, vp,
                                            ctypes.c_size_t]
        L.mec_conv_forward_host.restype = ci
        L.mec_last_launch_count.argtypes = []
        L.mec_last_launch_count.restype = ci
        L.mec_status_string.argtypes = [ci]
        L.mec_status_string.restype = ctypes.c_char_p
        L.mec_last_error_message.argtypes = []
        L.mec_last_error_message.restype = ctypes.c_char_p
        L.mec_abi_version.argtypes = []
        L.mec_abi_version.restype = ci
        L.mec_synth_fill.argtypes = [vp, i64, ctypes.c_uint64, ci, ctypes.c_uint64, ci, ci, vp]
        L.mec_synth_fill.restype = ci
        L.mec_l2_flush.argtypes = [vp, ctypes.c_size_t, vp]
        L.mec_l2_flush.restype = ci
        _lib = L
        return _lib


class MecError(RuntimeError):
    def __init__(self, status: int, where: str):
        L = lib()
        msg = L.mec_status_string(status).decode()
        detail = L.mec_last_error_message().decode() if status == MEC_ERR_CUDA else ""
        super().__init__(f"{where}: {msg} {detail}".strip())
        self.status = status


def check(status: int, where: str) -> None:
    if status != MEC_OK:
        raise MecError(status, where)
