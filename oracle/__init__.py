"""CPU oracle for MEC (arXiv 1706.06873) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It is a
ctypes wrapper over ``mec_oracle.c`` (plain C11, fp64 accumulation, no BLAS),
compiled with gcc.  It shares no code with ``paper_1706_06873_b200`` (the
CUDA path); neither imports the other.  Every function cites the PAPER.md
passage it follows (``P:<line>``); the readings of ambiguous passages are
listed in DESIGN.md section 3.

Parity status of every exported function (the pins live in
tests/test_oracle_pins.py; none of them re-calls the oracle's own formula):
  out_dims        -- Eq.1; Fig.1 caption (7,3,1 -> 5); Table 3 cv4 (floor)
  elems_L_mec,
  elems_L_im2col  -- Fig.1/Fig.2 sizes (25x9, 5x21); Table 3 MEM column; Eq.4
  elems_O         -- the #O > #L refusal cases of Alg.2 l.8 (cv3, cv7)
  select_path     -- Alg.2 l.8 evaluated by hand for the BASELINE configs,
                     inclusive threshold
  direct_conv     -- ramp closed form; torch.nn.functional.conv2d (fp64);
                     1x1 == GEMM; k == i == dot products
  im2col          -- Fig.1(b) 25x9; numpy matmul of it == torch conv2d
  lower           -- Fig.2 partitions A=I[0:7,0:3], B=I[0:7,1:4];
                     numpy sliding windows; horizontal-redundancy invariant;
                     1x1 == transpose
  vanilla_mec     -- == direct conv on Fig.1 shapes; P/Q partitions
  conv_solA/solB,
  mec             -- == torch conv2d (fp64) on random tiny shapes; A == B
No function is "parity unpinned".  (Round 2 removed an unused plain matmul
helper that had no pin of its own.)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mec_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile mec_oracle.c into liboracle.so with gcc (no GPU needed)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mec_oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
             "-o", tmp, _SRC]
        )
        os.replace(tmp, _SO)
    return _SO


class Shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("i_n", "i_h", "i_w", "i_c", "k_h", "k_w", "k_c")]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            P = ctypes.POINTER
            dp = P(ctypes.c_double)
            sp = P(Shape)
            i64p = P(ctypes.c_int64)
            lib.mec_oracle_out_dims.argtypes = [sp, ctypes.c_int, ctypes.c_int, i64p, i64p]
            for f in ("mec_oracle_elems_L_mec", "mec_oracle_elems_L_im2col", "mec_oracle_elems_O"):
                getattr(lib, f).argtypes = [sp, ctypes.c_int, ctypes.c_int]
                getattr(lib, f).restype = ctypes.c_int64
            lib.mec_oracle_select_path.argtypes = [sp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
            lib.mec_oracle_direct_conv.argtypes = [dp, dp, dp, sp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
            lib.mec_oracle_im2col.argtypes = [dp, dp, sp, ctypes.c_int, ctypes.c_int]
            lib.mec_oracle_lower.argtypes = [ctypes.c_void_p, ctypes.c_void_p, sp, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_size_t]
            lib.mec_oracle_vanilla_mec.argtypes = [dp, dp, dp] + [ctypes.c_int64] * 4 + [ctypes.c_int] * 2
            lib.mec_oracle_conv_solA.argtypes = [dp, dp, dp, sp, ctypes.c_int, ctypes.c_int]
            lib.mec_oracle_conv_solB.argtypes = [dp, dp, dp, sp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
            lib.mec_oracle_mec.argtypes = [dp, dp, dp, sp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, P(ctypes.c_int)]
            _lib = lib
    return _lib


def _shape(shape) -> Shape:
    """shape: dict or 7-tuple (i_n, i_h, i_w, i_c, k_h, k_w, k_c) -- Table 1 symbols."""
    if isinstance(shape, dict):
        return Shape(*(int(shape[k]) for k in ("i_n", "i_h", "i_w", "i_c", "k_h", "k_w", "k_c")))
    return Shape(*(int(v) for v in shape))


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def out_dims(shape, s_h: int, s_w: int):
    """Eq. (1), floor (reading Q1). Returns (o_h, o_w); raises on invalid."""
    oh, ow = ctypes.c_int64(), ctypes.c_int64()
    if _load().mec_oracle_out_dims(ctypes.byref(_shape(shape)), s_h, s_w,
                                   ctypes.byref(oh), ctypes.byref(ow)):
        raise ValueError("invalid convolution shape")
    return oh.value, ow.value


def elems_L_mec(shape, s_h, s_w) -> int:
    """#L of MEC = i_n o_w i_h k_w i_c (Table 1; Alg.2 l.2)."""
    return _load().mec_oracle_elems_L_mec(ctypes.byref(_shape(shape)), s_h, s_w)


def elems_L_im2col(shape, s_h, s_w) -> int:
    """#L of im2col = i_n o_h o_w k_h k_w i_c (Eq. 2; reading Q2)."""
    return _load().mec_oracle_elems_L_im2col(ctypes.byref(_shape(shape)), s_h, s_w)


def elems_O(shape, s_h, s_w) -> int:
    """#O = i_n o_h o_w k_c (Alg.2 l.1)."""
    return _load().mec_oracle_elems_O(ctypes.byref(_shape(shape)), s_h, s_w)


def select_path(shape, s_h, s_w, T: int = 100) -> int:
    """Alg.2 l.8: 1 = Solution A iff o_w <= T and #O <= #L, else 2 = Solution B."""
    return _load().mec_oracle_select_path(ctypes.byref(_shape(shape)), s_h, s_w, T)


def _check(rc):
    if rc == -2:
        raise ValueError("Solution A unavailable: #O > #L (P:211)")
    if rc != 0:
        raise ValueError(f"oracle call failed ({rc})")


def direct_conv(I: np.ndarray, K: np.ndarray, s_h: int, s_w: int, n_threads: int = 1) -> np.ndarray:
    """Direct convolution (Fig. 1(a)).  I: (i_n,i_h,i_w,i_c), K: (k_h,k_w,i_c,k_c), fp64."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    shp = (*I.shape, K.shape[0], K.shape[1], K.shape[3])
    assert K.shape[2] == I.shape[3]
    oh, ow = out_dims(shp, s_h, s_w)
    O = np.empty((I.shape[0], oh, ow, K.shape[3]), dtype=np.float64)
    _check(_load().mec_oracle_direct_conv(_dptr(I), _dptr(K), _dptr(O),
                                          ctypes.byref(_shape(shp)), s_h, s_w, n_threads))
    return O


def im2col(I: np.ndarray, k_h: int, k_w: int, s_h: int, s_w: int) -> np.ndarray:
    """im2col lowered matrix (Fig. 1(b), Eq. 2): (i_n o_h o_w) x (k_h k_w i_c)."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    shp = (*I.shape, k_h, k_w, 1)
    oh, ow = out_dims(shp, s_h, s_w)
    C = np.empty((I.shape[0] * oh * ow, k_h * k_w * I.shape[3]), dtype=np.float64)
    _check(_load().mec_oracle_im2col(_dptr(I), _dptr(C), ctypes.byref(_shape(shp)), s_h, s_w))
    return C


def lower(I: np.ndarray, k_h: int, k_w: int, s_h: int, s_w: int) -> np.ndarray:
    """MEC lowering (Alg.2 l.3-6).  Works on any dtype as a bit copy;
    returns L with shape (i_n, o_w, i_h, k_w, i_c) and I's dtype."""
    I = np.ascontiguousarray(I)
    shp = (*I.shape, k_h, k_w, 1)
    oh, ow = out_dims(shp, s_h, s_w)
    L = np.empty((I.shape[0], ow, I.shape[1], k_w, I.shape[3]), dtype=I.dtype)
    _check(_load().mec_oracle_lower(I.ctypes.data, L.ctypes.data, ctypes.byref(_shape(shp)),
                                    s_h, s_w, I.dtype.itemsize))
    return L


def vanilla_mec(I2: np.ndarray, K2: np.ndarray, s_h: int, s_w: int) -> np.ndarray:
    """Algorithm 1, i_n = i_c = k_c = 1.  I2: (i_h,i_w), K2: (k_h,k_w)."""
    I2 = np.ascontiguousarray(I2, dtype=np.float64)
    K2 = np.ascontiguousarray(K2, dtype=np.float64)
    i_h, i_w = I2.shape
    k_h, k_w = K2.shape
    oh, ow = (i_h - k_h) // s_h + 1, (i_w - k_w) // s_w + 1
    O = np.empty((oh, ow), dtype=np.float64)
    _check(_load().mec_oracle_vanilla_mec(_dptr(I2), _dptr(K2), _dptr(O), i_h, i_w, k_h, k_w, s_h, s_w))
    return O


def conv_solA(I, K, s_h, s_w) -> np.ndarray:
    """Alg.2 Solution A (l.9-19) literally, incl. 'Copy L = O' and the transpose."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    shp = (*I.shape, K.shape[0], K.shape[1], K.shape[3])
    oh, ow = out_dims(shp, s_h, s_w)
    O = np.empty((I.shape[0], oh, ow, K.shape[3]), dtype=np.float64)
    _check(_load().mec_oracle_conv_solA(_dptr(I), _dptr(K), _dptr(O), ctypes.byref(_shape(shp)), s_h, s_w))
    return O


def conv_solB(I, K, s_h, s_w, n_threads: int = 1) -> np.ndarray:
    """Alg.2 Solution B (l.20-25): per-image window GEMMs."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    shp = (*I.shape, K.shape[0], K.shape[1], K.shape[3])
    oh, ow = out_dims(shp, s_h, s_w)
    O = np.empty((I.shape[0], oh, ow, K.shape[3]), dtype=np.float64)
    _check(_load().mec_oracle_conv_solB(_dptr(I), _dptr(K), _dptr(O), ctypes.byref(_shape(shp)),
                                        s_h, s_w, n_threads))
    return O


def mec(I, K, s_h, s_w, T: int = 100, n_threads: int = 1):
    """Algorithm 2 end to end.  Returns (O, path) with path 1=A, 2=B."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    shp = (*I.shape, K.shape[0], K.shape[1], K.shape[3])
    oh, ow = out_dims(shp, s_h, s_w)
    O = np.empty((I.shape[0], oh, ow, K.shape[3]), dtype=np.float64)
    path = ctypes.c_int()
    _check(_load().mec_oracle_mec(_dptr(I), _dptr(K), _dptr(O), ctypes.byref(_shape(shp)),
                                  s_h, s_w, T, n_threads, ctypes.byref(path)))
    return O, path.value
