"""Python binding of the MEC C ABI (include/mec.h) -- argument marshalling only.

Every step of the computation runs in libmec.so's CUDA kernels on the
caller's current torch CUDA stream.  torch supplies device memory and the
stream; nothing here computes.  Inputs must be CUDA tensors: there is no CPU
fallback, and a missing library raises.

Layouts follow the paper's Table 1: I (i_n, i_h, i_w, i_c) NHWC,
K (k_h, k_w, i_c, k_c), O (i_n, o_h, o_w, k_c), L (i_n, o_w, i_h, k_w, i_c).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (MEC_DTYPE_BF16, MEC_DTYPE_TF32, MEC_PATH_AUTO, MEC_PATH_FASTEST, MEC_PATH_FUSED,  # noqa: F401
                   MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B, MEC_SOLA_FIX_EPILOGUE,
                   MEC_SOLA_FIX_LITERAL, MEC_SOLA_FIX_NONE, MEC_DEFAULT_T, MecError)

PATH_NAMES = {MEC_PATH_SOLUTION_A: "solution_A_batch_folded", MEC_PATH_SOLUTION_B: "solution_B_per_image",
              MEC_PATH_FUSED: "fused"}


def _shape(i_n, i_h, i_w, i_c, k_h, k_w, k_c) -> _lib.MecShape:
    return _lib.MecShape(int(i_n), int(i_h), int(i_w), int(i_c), int(k_h), int(k_w), int(k_c))


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return MEC_DTYPE_BF16
    if dt == torch.float32:
        return MEC_DTYPE_TF32
    raise TypeError(f"MEC supports bfloat16 and float32 (tf32 math), got {dt}")


def _stream(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (MEC has no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def out_dims(i_h, i_w, k_h, k_w, s_h, s_w):
    """Eq. (1), P:43 (floor)."""
    oh, ow = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().mec_out_dims(ctypes.byref(_shape(1, i_h, i_w, 1, k_h, k_w, 1)), s_h, s_w,
                                       ctypes.byref(oh), ctypes.byref(ow)), "mec_out_dims")
    return oh.value, ow.value


def select_path(shape, s_h, s_w, T: int = MEC_DEFAULT_T) -> int:
    """Alg.2 l.8: MEC_PATH_SOLUTION_A or MEC_PATH_SOLUTION_B.  shape = 7-tuple."""
    r = _lib.lib().mec_select_path(ctypes.byref(_shape(*shape)), s_h, s_w, T)
    if r == MEC_PATH_AUTO:
        raise ValueError("invalid shape")
    return r


def lowered_elems(shape, s_h, s_w) -> int:
    return _lib.lib().mec_lowered_elems(ctypes.byref(_shape(*shape)), s_h, s_w)


def im2col_elems(shape, s_h, s_w) -> int:
    return _lib.lib().mec_im2col_elems(ctypes.byref(_shape(*shape)), s_h, s_w)


def workspace_bytes(shape, s_h, s_w, dtype: torch.dtype, pad_h: int = 0, pad_w: int = 0, **opts) -> int:
    """mec_workspace_bytes (or _ex with pads / options such as path, gemm_kernel, split_k)."""
    if pad_h == 0 and pad_w == 0 and not opts:
        return _lib.lib().mec_workspace_bytes(ctypes.byref(_shape(*shape)), s_h, s_w, dtype_code(dtype))
    opt = _lib.MecOptions()
    _lib.lib().mec_options_init(ctypes.byref(opt))
    opt.pad_h, opt.pad_w = int(pad_h), int(pad_w)
    for k, v in opts.items():
        setattr(opt, k, int(v))
    return _lib.lib().mec_workspace_bytes_ex(ctypes.byref(_shape(*shape)), s_h, s_w, dtype_code(dtype),
                                             ctypes.byref(opt))


def lower(I: torch.Tensor, k_h: int, k_w: int, s_h: int, s_w: int, out: torch.Tensor | None = None,
          pad_h: int = 0, pad_w: int = 0):
    """mec_lower / mec_lower_padded: L = compact lowering of I (Alg.2 l.3-6), dense
    (i_n, o_w, i_h', k_w, i_c) of the input zero-padded by pad_h / pad_w (i_h' = i_h + 2 pad_h)."""
    _cuda(I, "I")
    i_n, i_h, i_w, i_c = I.shape
    hp, wp = i_h + 2 * pad_h, i_w + 2 * pad_w
    o_h, o_w = out_dims(hp, wp, k_h, k_w, s_h, s_w)
    if out is None:
        out = torch.empty((i_n, o_w, hp, k_w, i_c), dtype=I.dtype, device=I.device)
    _cuda(out, "L")
    assert out.dtype == I.dtype and out.numel() == i_n * o_w * hp * k_w * i_c
    _lib.check(_lib.lib().mec_lower_padded(I.data_ptr(), out.data_ptr(),
                                           ctypes.byref(_shape(i_n, i_h, i_w, i_c, k_h, k_w, 1)),
                                           s_h, s_w, int(pad_h), int(pad_w), dtype_code(I.dtype), _stream(I)),
               "mec_lower_padded")
    return out


def lower_pitched(I: torch.Tensor, k_h: int, k_w: int, s_h: int, s_w: int, pitch: int | None = None):
    """mec_lower_pitched: the conv path's lowered layout -- i_n o_w rows of L
    (i_h k_w i_c elements each, Alg.2 l.9) at a row pitch of `pitch` elements
    (default: rounded up to 16 bytes, as the conv path uses).  Returns the
    (i_n o_w, pitch) buffer; columns past i_h k_w i_c are unspecified."""
    _cuda(I, "I")
    i_n, i_h, i_w, i_c = I.shape
    o_h, o_w = out_dims(i_h, i_w, k_h, k_w, s_h, s_w)
    cols = i_h * k_w * i_c
    if pitch is None:
        v = 16 // I.element_size()
        pitch = (cols + v - 1) // v * v
    out = torch.empty((i_n * o_w, pitch), dtype=I.dtype, device=I.device)
    _lib.check(_lib.lib().mec_lower_pitched(I.data_ptr(), out.data_ptr(),
                                            ctypes.byref(_shape(i_n, i_h, i_w, i_c, k_h, k_w, 1)),
                                            s_h, s_w, int(pitch), dtype_code(I.dtype), _stream(I)),
               "mec_lower_pitched")
    return out


def conv_forward(I: torch.Tensor, K: torch.Tensor, s_h: int, s_w: int, out: torch.Tensor | None = None,
                 path: int = MEC_PATH_AUTO, T: int = MEC_DEFAULT_T, sola_fix: int = MEC_SOLA_FIX_EPILOGUE,
                 workspace: torch.Tensor | None = None, stage_events=None, return_path: bool = False,
                 rows_per_tile: int = 0, pad_h: int = 0, pad_w: int = 0, return_gemm: bool = False,
                 gemm_kernel: int = 0, split_k: int = 0, return_split: bool = False):
    """mec_conv_forward_ex: O = MEC(I, K, s) (Algorithm 2), O in n-h-w-c
    (or h-n-w-c with sola_fix=MEC_SOLA_FIX_NONE when Solution A runs).  pad_h / pad_w:
    zero padding applied virtually inside the lowering (never materialised).
    return_path / return_gemm / return_split: also return the path that ran (1 = A, 2 = B,
    3 = fused) / the window-GEMM kernel that ran (1 = one window per tile, 2 = h-sweep,
    3 = CTA pair) / the CTA-pair kernel's split-K count.  gemm_kernel forces the kernel
    (0 = automatic), split_k the CTA-pair kernel's K ranges (0 = automatic)."""
    _cuda(I, "I")
    _cuda(K, "K")
    if K.dtype != I.dtype:
        raise TypeError("I and K must have the same dtype")
    i_n, i_h, i_w, i_c = I.shape
    k_h, k_w, k_ci, k_c = K.shape
    if k_ci != i_c:
        raise ValueError("K's third extent must equal i_c (Table 1)")
    o_h, o_w = out_dims(i_h + 2 * pad_h, i_w + 2 * pad_w, k_h, k_w, s_h, s_w)
    if out is None:
        out = torch.empty((i_n, o_h, o_w, k_c), dtype=I.dtype, device=I.device)
    _cuda(out, "O")
    assert out.dtype == I.dtype and out.numel() == i_n * o_h * o_w * k_c
    opt = _lib.MecOptions()
    _lib.lib().mec_options_init(ctypes.byref(opt))
    opt.path, opt.T, opt.sola_fix = int(path), int(T), int(sola_fix)
    opt.rows_per_tile = int(rows_per_tile)
    opt.pad_h, opt.pad_w = int(pad_h), int(pad_w)
    opt.gemm_kernel, opt.split_k = int(gemm_kernel), int(split_k)
    if workspace is not None:
        _cuda(workspace, "workspace")
        opt.workspace = workspace.data_ptr()
        opt.workspace_bytes = workspace.numel() * workspace.element_size()
    if stage_events is not None:
        for i, ev in enumerate(stage_events[:4]):
            opt.stage_events[i] = ev.cuda_event if ev is not None else None
    st = _lib.lib().mec_conv_forward_ex(I.data_ptr(), K.data_ptr(), out.data_ptr(),
                                        ctypes.byref(_shape(i_n, i_h, i_w, i_c, k_h, k_w, k_c)),
                                        s_h, s_w, dtype_code(I.dtype), _stream(I), ctypes.byref(opt))
    _lib.check(st, "mec_conv_forward")
    extra = (([opt.selected_path] if return_path else []) + ([opt.selected_gemm] if return_gemm else [])
             + ([opt.selected_split] if return_split else []))
    return (out, *extra) if extra else out


def host_scratch_bytes(i_n, i_h, i_w, i_c, k_h, k_w, k_c, s_h, s_w, dtype, n_chunks,
                       pad_h: int = 0, pad_w: int = 0) -> int:
    """mec_host_scratch_bytes: device scratch of conv_forward_host for this problem."""
    opt = _lib.MecOptions()
    _lib.lib().mec_options_init(ctypes.byref(opt))
    opt.pad_h, opt.pad_w = int(pad_h), int(pad_w)
    return int(_lib.lib().mec_host_scratch_bytes(ctypes.byref(_shape(i_n, i_h, i_w, i_c, k_h, k_w, k_c)),
                                                 s_h, s_w, dtype_code(dtype), ctypes.byref(opt),
                                                 int(n_chunks)))


def auto_chunks(i_n: int, bytes_in_out: int) -> int:
    """Image chunks of the host-buffer call: ~48 MB of copies per chunk, 4 to 16
    chunks (measured on B200 + PCIe gen5: VGG conv1_2 b64, 815 MB per call:
    1/2/4/8/16 chunks 15.0/11.7/10.1/9.6/9.2 ms; AlexNet conv1 b32, 29 MB:
    4 chunks best, 0.50 ms, 8 chunks 0.58 ms -- each copy pair costs ~7 us)."""
    return max(1, min(i_n, max(4, min(16, -(-bytes_in_out // (48 << 20))))))


def conv_forward_host(I_h: torch.Tensor, K_h: torch.Tensor, s_h: int, s_w: int, out: torch.Tensor | None = None,
                      n_chunks: int | None = None, path: int = MEC_PATH_AUTO, T: int = MEC_DEFAULT_T,
                      sola_fix: int = MEC_SOLA_FIX_EPILOGUE, scratch: torch.Tensor | None = None,
                      pad_h: int = 0, pad_w: int = 0, device=None, return_path: bool = False):
    """mec_conv_forward_host: O = MEC(I, K, s) on HOST tensors (pinned for asynchronous copies):
    the copies in and out run inside the call, pipelined over n_chunks chunks of images
    (None: auto_chunks).
    Enqueued on the current stream of `device` (default: the current CUDA device); O is
    complete once that stream is synchronised.  scratch: a device uint8 tensor of at least
    host_scratch_bytes(...) bytes (None = the library's stream-ordered pool)."""
    for t, n in ((I_h, "I"), (K_h, "K")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{n} must be a contiguous HOST tensor")
    if K_h.dtype != I_h.dtype:
        raise TypeError("I and K must have the same dtype")
    i_n, i_h, i_w, i_c = I_h.shape
    k_h, k_w, k_ci, k_c = K_h.shape
    if k_ci != i_c:
        raise ValueError("K's third extent must equal i_c (Table 1)")
    o_h, o_w = out_dims(i_h + 2 * pad_h, i_w + 2 * pad_w, k_h, k_w, s_h, s_w)
    if out is None:
        out = torch.empty((i_n, o_h, o_w, k_c), dtype=I_h.dtype, pin_memory=True)
    if out.is_cuda or not out.is_contiguous():
        raise ValueError("O must be a contiguous HOST tensor")
    assert out.dtype == I_h.dtype and out.numel() == i_n * o_h * o_w * k_c
    if n_chunks is None:
        n_chunks = auto_chunks(i_n, (I_h.numel() + out.numel()) * I_h.element_size())
    opt = _lib.MecOptions()
    _lib.lib().mec_options_init(ctypes.byref(opt))
    opt.path, opt.T, opt.sola_fix = int(path), int(T), int(sola_fix)
    opt.pad_h, opt.pad_w = int(pad_h), int(pad_w)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    sp, sb = None, 0
    if scratch is not None:
        _cuda(scratch, "scratch")
        sp, sb = scratch.data_ptr(), scratch.numel() * scratch.element_size()
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        st = _lib.lib().mec_conv_forward_host(I_h.data_ptr(), K_h.data_ptr(), out.data_ptr(),
                                              ctypes.byref(_shape(i_n, i_h, i_w, i_c, k_h, k_w, k_c)),
                                              s_h, s_w, dtype_code(I_h.dtype), stream, ctypes.byref(opt),
                                              int(n_chunks), sp, sb)
    _lib.check(st, "mec_conv_forward_host")
    # The copies read I_h / K_h and write out asynchronously: keep the tensors
    # (and the scratch) alive until the stream passes an event recorded after
    # the call, so a temporary argument (x.pin_memory()) is not freed -- and
    # its pinned block reused -- while a copy still reads it.
    with torch.cuda.device(dev):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
    _keep_alive(ev, (I_h, K_h, out, scratch))
    return (out, opt.selected_path) if return_path else out


_PENDING: list = []  # (event, tensors) of host-buffer calls still in flight


def _keep_alive(ev, refs) -> None:
    """Hold `refs` until `ev` has completed; completed entries are dropped here."""
    _PENDING[:] = [(e, r) for e, r in _PENDING if not e.query()]
    _PENDING.append((ev, refs))


def maxpool(X: torch.Tensor, p_h: int, p_w: int, s_h: int, s_w: int, hnwc: bool = False,
            out: torch.Tensor | None = None) -> torch.Tensor:
    """mec_maxpool: max pooling of a conv output X, given as (i_n, h, w, c) n-h-w-c or, with
    hnwc=True, as Solution A's (h, i_n, w, c) h-n-w-c; returns (i_n, o_h, o_w, c) n-h-w-c."""
    _cuda(X, "X")
    if hnwc:
        h, i_n, w, c = X.shape
    else:
        i_n, h, w, c = X.shape
    o_h, o_w = (h - p_h) // s_h + 1, (w - p_w) // s_w + 1
    if out is None:
        out = torch.empty((i_n, o_h, o_w, c), dtype=X.dtype, device=X.device)
    _cuda(out, "Y")
    _lib.check(_lib.lib().mec_maxpool(X.data_ptr(), out.data_ptr(), i_n, h, w, c, p_h, p_w, s_h, s_w,
                                      _lib.MEC_LAYOUT_HNWC if hnwc else _lib.MEC_LAYOUT_NHWC,
                                      dtype_code(X.dtype), _stream(X)), "mec_maxpool")
    return out


def last_launch_count() -> int:
    return _lib.lib().mec_last_launch_count()


def synth_fill(t: torch.Tensor, seed: int, tensor_id: int, kind: int, index_offset: int = 0) -> torch.Tensor:
    """Device-side counter-based generator (include/mec_synth.h) into tensor t."""
    _cuda(t, "t")
    _lib.check(_lib.lib().mec_synth_fill(t.data_ptr(), t.numel(), seed, tensor_id, index_offset, kind,
                                         dtype_code(t.dtype), _stream(t)), "mec_synth_fill")
    return t


def l2_flush(scratch: torch.Tensor) -> None:
    _cuda(scratch, "scratch")
    _lib.check(_lib.lib().mec_l2_flush(scratch.data_ptr(), scratch.numel() * scratch.element_size(),
                                       _stream(scratch)), "mec_l2_flush")
