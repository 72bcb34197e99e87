"""CPU-only checks of the C ABI: libmec.so loads, exports every symbol the
headers declare, and its host-only entry points (planning, Eq. 1, the T rule,
closed-form sizes, argument validation) behave as include/mec.h states.
No compute call is made (there is no GPU here)."""
import ctypes
import re

import pytest

import oracle
from paper_1706_06873_b200 import _lib, mec
from synth.configs import CONFIGS, TABLE2
from mec_testutil import ROOT


def header_symbols():
    syms = set()
    for h in ("mec.h", "mec_synth.h"):
        txt = open(f"{ROOT}/include/{h}").read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(mec_[a-z0-9_]+)\s*\(", txt):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_symbols()
    assert declared == set(_lib.EXPORTED)
    for s in declared:
        assert hasattr(L, s), s
    assert L.mec_abi_version() == 6


def test_status_strings():
    L = _lib.lib()
    for code, name in [(0, "MEC_OK"), (1, "MEC_ERR_INVALID_ARG"), (2, "MEC_ERR_UNSUPPORTED"),
                       (3, "MEC_ERR_MISALIGNED"), (4, "MEC_ERR_CUDA"), (5, "MEC_ERR_NO_MEMORY")]:
        assert L.mec_status_string(code).decode() == name


def shape7(c):
    return (c["i_n"], c["i_h"], c["i_w"], c["i_c"], c["k_h"], c["k_w"], c["k_c"])


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_plan_matches_oracle_for_every_config(name):
    c = CONFIGS[name]
    shp = shape7(c)
    s_h, s_w = c["s_h"], c["s_w"]
    assert mec.out_dims(c["i_h"], c["i_w"], c["k_h"], c["k_w"], s_h, s_w) == oracle.out_dims(shp, s_h, s_w)
    assert mec.select_path(shp, s_h, s_w) == oracle.select_path(shp, s_h, s_w, 100)
    assert mec.lowered_elems(shp, s_h, s_w) == oracle.elems_L_mec(shp, s_h, s_w)
    assert mec.im2col_elems(shp, s_h, s_w) == oracle.elems_L_im2col(shp, s_h, s_w)


@pytest.mark.parametrize("T", [1, 50, 100, 200, 1000])
def test_select_path_threshold_sweep(T):
    for name, (i_h, i_w, i_c, k_h, k_w, k_c, s) in TABLE2.items():
        shp = (8, i_h, i_w, i_c, k_h, k_w, k_c)
        assert mec.select_path(shp, s, s, T) == oracle.select_path(shp, s, s, T), name


def test_workspace_is_lowered_size_not_im2col():
    import torch

    for name, c in CONFIGS.items():
        shp = shape7(c)
        for dt, elt in ((torch.bfloat16, 2), (torch.float32, 4)):
            ws = mec.workspace_bytes(shp, c["s_h"], c["s_w"], dt)
            n_l = oracle.elems_L_mec(shp, c["s_h"], c["s_w"])
            o_h, o_w = oracle.out_dims(shp, c["s_h"], c["s_w"])
            pitch = -(-(c["i_h"] * c["k_w"] * c["i_c"]) // (16 // elt)) * (16 // elt)
            L_pitched = c["i_n"] * o_w * pitch * elt
            assert ws >= n_l * elt and ws >= L_pitched
            # only pitch padding (rows rounded up to at most 32 bytes, the window
            # GEMM's box alignment; strips padded by at most 15%)
            # + the prepared K (at most 8 shifted copies) + alignment on top of L
            pitch32 = -(-(c["i_h"] * c["k_w"] * c["i_c"]) // (32 // elt)) * (32 // elt)
            L_pitched32 = int(c["i_n"] * o_w * (pitch32 * 1.15 + 32 // elt) * elt)
            kt = 8 * (-(-c["k_c"] // 16) * 16 + 256) * (-(-(c["k_h"] * c["k_w"] * c["i_c"]) // 64) * 64 + 64) * elt
            assert ws <= L_pitched32 + kt + 4096, name
            if c["k_h"] > c["s_h"] and (c["i_h"] - c["k_h"]) % c["s_h"] == 0:
                # the lowered buffer itself is smaller than im2col's (Eq. 4); on the batched
                # configs so is the whole workspace
                assert L_pitched < oracle.elems_L_im2col(shp, c["s_h"], c["s_w"]) * elt, name
                if c["i_n"] >= 32:
                    assert ws < oracle.elems_L_im2col(shp, c["s_h"], c["s_w"]) * elt, name


@pytest.mark.parametrize("bad", [
    (0, 7, 7, 1, 3, 3, 1), (1, 7, 7, 0, 3, 3, 1), (1, 7, 7, 1, 3, 3, 0), (1, 2, 7, 1, 3, 3, 1),
    (1, 7, 2, 1, 3, 3, 1), (1, 7, 7, 1, 0, 3, 1), (-1, 7, 7, 1, 3, 3, 1),
])
def test_invalid_shapes_rejected_host_side(bad):
    L = _lib.lib()
    s = _lib.MecShape(*bad)
    oh, ow = ctypes.c_int64(), ctypes.c_int64()
    assert L.mec_out_dims(ctypes.byref(s), 1, 1, ctypes.byref(oh), ctypes.byref(ow)) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_workspace_bytes(ctypes.byref(s), 1, 1, 0) == 0
    assert L.mec_select_path(ctypes.byref(s), 1, 1, 100) == 0
    assert L.mec_lowered_elems(ctypes.byref(s), 1, 1) == -1
    # validation happens before any device work: NULL / fake pointers are never touched
    assert L.mec_lower(None, None, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_conv_forward(None, None, None, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_INVALID_ARG


def test_argument_validation_without_device_work():
    L = _lib.lib()
    s = _lib.MecShape(1, 7, 7, 1, 3, 3, 1)
    # stride < 1, bad dtype
    assert L.mec_lower(16, 32, ctypes.byref(s), 0, 1, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_lower(16, 32, ctypes.byref(s), 1, 1, 7, None) == _lib.MEC_ERR_INVALID_ARG
    # NULL pointers
    assert L.mec_lower(None, 32, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_conv_forward(16, None, 48, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_INVALID_ARG
    # misaligned (checked before anything touches the pointers)
    assert L.mec_lower(18, 32, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_MISALIGNED
    assert L.mec_conv_forward(16, 34, 48, ctypes.byref(s), 1, 1, 0, None) == _lib.MEC_ERR_MISALIGNED
    # bad enum in options
    opt = _lib.MecOptions()
    L.mec_options_init(ctypes.byref(opt))
    assert (opt.path, opt.T, opt.sola_fix) == (0, 100, 0)
    opt.path = 9
    assert L.mec_conv_forward_ex(16, 32, 48, ctypes.byref(s), 1, 1, 0, None, ctypes.byref(opt)) == \
        _lib.MEC_ERR_INVALID_ARG
    # forced fused path on a shape neither fused variant takes (k_c > 256: two N tiles,
    # i_c elt not a multiple of 128 B) -- rejected host-side
    s3 = _lib.MecShape(1, 7, 7, 1, 3, 3, 300)
    L.mec_options_init(ctypes.byref(opt))
    opt.path = _lib.MEC_PATH_FUSED
    assert L.mec_conv_forward_ex(16, 32, 48, ctypes.byref(s3), 1, 1, 0, None, ctypes.byref(opt)) == \
        _lib.MEC_ERR_UNSUPPORTED
    # Solution A's literal format fix needs #L >= #O: 1x6x6x1, 3x3x8 -> #O 128 > #L 72
    s2 = _lib.MecShape(1, 6, 6, 1, 3, 3, 8)
    L.mec_options_init(ctypes.byref(opt))
    opt.path, opt.sola_fix = _lib.MEC_PATH_SOLUTION_A, _lib.MEC_SOLA_FIX_LITERAL
    assert L.mec_conv_forward_ex(16, 32, 48, ctypes.byref(s2), 1, 1, 0, None, ctypes.byref(opt)) == \
        _lib.MEC_ERR_UNSUPPORTED
    # workspace too small
    L.mec_options_init(ctypes.byref(opt))
    opt.workspace, opt.workspace_bytes = 4096, 16
    assert L.mec_conv_forward_ex(16, 32, 48, ctypes.byref(s), 1, 1, 0, None, ctypes.byref(opt)) == \
        _lib.MEC_ERR_NO_MEMORY
    # mec_lower_pitched: pitch below one L row, pitch not 16-byte granular, misaligned L
    assert L.mec_lower_pitched(16, 32, ctypes.byref(s), 1, 1, 20, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_lower_pitched(16, 32, ctypes.byref(s), 1, 1, 21, 0, None) == _lib.MEC_ERR_MISALIGNED
    assert L.mec_lower_pitched(16, 40, ctypes.byref(s), 1, 1, 24, 0, None) == _lib.MEC_ERR_MISALIGNED
    # synth helper validation
    assert L.mec_synth_fill(None, 10, 1, 0, 0, 0, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_synth_fill(16, 10, 1, 0, 0, 5, 0, None) == _lib.MEC_ERR_INVALID_ARG
    assert L.mec_l2_flush(None, 10, None) == _lib.MEC_ERR_INVALID_ARG


def test_python_binding_refuses_cpu_tensors():
    import torch

    with pytest.raises(TypeError):
        mec.conv_forward(torch.zeros(1, 7, 7, 1), torch.zeros(3, 3, 1, 1), 1, 1)
    with pytest.raises(TypeError):
        mec.lower(torch.zeros(1, 7, 7, 1), 3, 3, 1, 1)


def test_product_package_does_not_import_oracle():
    import pathlib

    for p in pathlib.Path(f"{ROOT}/paper_1706_06873_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".h", ".cpp"):
            txt = p.read_text()
            assert "oracle" not in txt.replace("oracle/", "").lower() or "import oracle" not in txt, p
            assert "import oracle" not in txt and "from oracle" not in txt, p
            assert "mec_oracle" not in txt, p


def test_host_call_scratch_layout_and_validation():
    """mec_host_scratch_bytes / mec_conv_forward_host (ABI 4): the scratch holds K, a ring of
    min(3, chunks) I and O chunk slots and the workspace of one chunk; every argument error is
    returned before any device work (fake pointers are never touched)."""
    L = _lib.lib()
    bf = _lib.MEC_DTYPE_BF16
    shp = (32, 227, 227, 3, 11, 11, 96)
    s = _lib.MecShape(*shp)
    i_img, o_img, k_b = 227 * 227 * 3 * 2, 55 * 55 * 96 * 2, 11 * 11 * 3 * 96 * 2
    up = lambda x: (x + 1023) // 1024 * 1024  # noqa: E731
    for nch, per, slots in [(1, 32, 1), (2, 16, 2), (4, 8, 3), (5, 7, 3), (64, 1, 3)]:
        sub = _lib.MecShape(per, *shp[1:])
        wsb = L.mec_workspace_bytes(ctypes.byref(sub), 4, 4, bf)
        want = up(k_b) + slots * (up(i_img * per) + up(o_img * per)) + wsb + 1024
        assert L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, nch) == want, nch
    # n_chunks is clamped to [1, i_n]
    one = L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, 1)
    assert L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, 0) == one
    assert L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, -5) == one
    assert (L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, 1000)
            == L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, 32))
    bad = _lib.MecShape(1, 2, 2, 1, 3, 3, 1)
    assert L.mec_host_scratch_bytes(ctypes.byref(bad), 1, 1, bf, None, 1) == 0
    fake = ctypes.c_void_p(0x1000)
    opt = _lib.MecOptions()
    L.mec_options_init(ctypes.byref(opt))
    call = lambda sh, o, scr, nb, I=fake: L.mec_conv_forward_host(  # noqa: E731
        I, fake, fake, ctypes.byref(sh), 4, 4, bf, None, o, 4, scr, nb)
    assert call(s, ctypes.byref(opt), fake, 1 << 40, I=None) == _lib.MEC_ERR_INVALID_ARG
    assert call(bad, ctypes.byref(opt), fake, 1 << 40) == _lib.MEC_ERR_INVALID_ARG
    need = L.mec_host_scratch_bytes(ctypes.byref(s), 4, 4, bf, None, 4)
    assert call(s, ctypes.byref(opt), fake, need - 1) == _lib.MEC_ERR_NO_MEMORY
    assert call(s, ctypes.byref(opt), ctypes.c_void_p(0x1008), need) == _lib.MEC_ERR_MISALIGNED
    opt.sola_fix = _lib.MEC_SOLA_FIX_NONE
    assert call(s, ctypes.byref(opt), fake, need) == _lib.MEC_ERR_UNSUPPORTED
    opt.sola_fix, opt.path = _lib.MEC_SOLA_FIX_EPILOGUE, 7
    assert call(s, ctypes.byref(opt), fake, need) == _lib.MEC_ERR_INVALID_ARG
