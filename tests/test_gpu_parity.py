"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Inputs come from the counter-based generator (synth/), evaluated on the host
for the oracle and uploaded for the GPU, so both sides see identical values.
Bars (BASELINE.json north_star):
  L                : bit-exact
  O, bf16          : max|O - O_ref| <= 2e-2 * max|O_ref|
  O, fp32 / tf32   : max|O - O_ref| <= 1e-3 * sqrt(k_h k_w i_c) * max|O_ref|
On the GRID kinds the inputs are exact in bf16 / tf32, so the GPU's only
error is fp32 accumulation order (+ the bf16 rounding of O); the tests also
check that much tighter bound.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1706_06873_b200 import mec
from paper_1706_06873_b200._lib import (MEC_PATH_FUSED, MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B, MEC_SOLA_FIX_EPILOGUE,
                                        MEC_SOLA_FIX_LITERAL, MEC_SOLA_FIX_NONE, MecError)

pytestmark = pytest.mark.gpu

TDT = {"bf16": torch.bfloat16, "tf32": torch.float32, "fp32": torch.float32}


def make_inputs(shape, dtype, seed, kind=None, n_begin=0):
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
    if kind is None:
        kind = synth.KIND_GRID8 if dtype == "bf16" else synth.KIND_GRID11
    cfg = dict(i_h=i_h, i_w=i_w, i_c=i_c, k_h=k_h, k_w=k_w, k_c=k_c)
    I = synth.input_images(cfg, n_begin, i_n, kind, seed)
    K = synth.kernel_tensor(cfg, kind, seed)
    return I, K


def to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(TDT[dtype])


def tol(dtype, kdim, ref):
    m = float(np.abs(ref).max()) if ref.size else 0.0
    return (2e-2 if dtype == "bf16" else 1e-3 * math.sqrt(kdim)) * max(m, 1e-30)


def check_O(O_gpu, ref, dtype, kdim, tight=True):
    got = O_gpu.float().cpu().numpy().astype(np.float64)
    assert got.shape == ref.shape
    err = float(np.abs(got - ref).max())
    bar = tol(dtype, kdim, ref)
    assert err <= bar, f"max abs err {err} > {bar}"
    if tight:
        # exact-grid inputs: only fp32 accumulation error (grows ~ sqrt(kdim) ulps) and,
        # for bf16, one RN rounding of O (<= 2^-8 |O|: 8 significant bits)
        m = float(np.abs(ref).max())
        acc = 2e-6 * math.sqrt(kdim) * m
        tight_bar = (2.0 ** -8 * m + acc if dtype == "bf16" else acc) + 1e-6
        assert err <= tight_bar, f"max abs err {err} > tight {tight_bar}"
    return err


SMALL = [
    # (i_n, i_h, i_w, i_c, k_h, k_w, k_c), s_h, s_w
    ((1, 7, 7, 1, 3, 3, 1), 1, 1),        # C0 shapes
    ((2, 9, 11, 3, 3, 5, 8), 1, 2),       # tiny, k_c 8
    ((3, 20, 17, 5, 4, 3, 24), 2, 1),     # k_c not multiple of 16, non-divisible stride
    ((2, 30, 30, 16, 3, 3, 40), 1, 1),
    ((4, 16, 40, 8, 5, 5, 64), 3, 2),     # s_h does not divide i_h - k_h
    ((2, 12, 12, 7, 2, 2, 17), 3, 3),     # s > k (unused input rows, reading Q5)
    ((1, 60, 70, 4, 1, 1, 32), 1, 1),     # 1x1
    ((2, 8, 9, 6, 8, 9, 48), 1, 1),       # k == i: o = 1
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(SMALL)))
def test_small_shapes_both_solutions(cuda_ok, case, dtype):
    shape, s_h, s_w = SMALL[case]
    I, K = make_inputs(shape, dtype, seed=1000 + case)
    ref = oracle.direct_conv(I, K, s_h, s_w)
    kdim = shape[4] * shape[5] * shape[3]
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    outs = {}
    for path in (MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B):
        O = mec.conv_forward(Id, Kd, s_h, s_w, path=path)
        torch.cuda.synchronize()
        check_O(O, ref, dtype, kdim)
        outs[path] = O
    # Both solutions share the mainloop: identical arithmetic per output element
    assert torch.equal(outs[MEC_PATH_SOLUTION_A], outs[MEC_PATH_SOLUTION_B])


def test_worked_example_ramp_exact(cuda_ok):
    # C0 (Fig. 1/2): ramp I[h,w] = 7h+w, K = ones -> O = 9(7h+w) + 72, exact in tf32/fp32
    I = np.array([[7 * h + w for w in range(7)] for h in range(7)], dtype=np.float32).reshape(1, 7, 7, 1)
    K = np.ones((3, 3, 1, 1), dtype=np.float32)
    expect = np.array([[9 * (7 * h + w) + 72 for w in range(5)] for h in range(5)], dtype=np.float32)
    for path in (0, MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B):
        O, chosen = mec.conv_forward(to_dev(I, "tf32"), to_dev(K, "tf32"), 1, 1, path=path, return_path=True)
        np.testing.assert_array_equal(O.cpu().numpy()[0, :, :, 0], expect)
        assert chosen == (path or MEC_PATH_SOLUTION_A)  # Alg.2 l.8: o_w 5 <= 100, #O 25 <= #L 105
    L = mec.lower(to_dev(I, "tf32"), 3, 3, 1, 1)
    assert tuple(L.shape) == (1, 5, 7, 3, 1)  # 5 x 21
    np.testing.assert_array_equal(L.cpu().numpy().reshape(5, 21)[1], I[0, :, 1:4, 0].reshape(-1))


@pytest.mark.parametrize("fix", [MEC_SOLA_FIX_EPILOGUE, MEC_SOLA_FIX_LITERAL, MEC_SOLA_FIX_NONE])
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_solution_A_format_fix_modes(cuda_ok, fix, dtype):
    shape, s = (5, 23, 21, 6, 3, 3, 24), 2
    I, K = make_inputs(shape, dtype, seed=77)
    ref = oracle.direct_conv(I, K, s, s)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    O = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, sola_fix=fix)
    torch.cuda.synchronize()
    if fix == MEC_SOLA_FIX_NONE:
        # h-n-w-c, the direct extension's format
        O = O.reshape(ref.shape[1], ref.shape[0], ref.shape[2], ref.shape[3]).permute(1, 0, 2, 3)
    check_O(O, ref, dtype, 54)
    base = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A)
    if fix != MEC_SOLA_FIX_NONE:
        assert torch.equal(O, base)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("name", ["cv1", "cv3", "cv5", "cv6", "cv9", "cv12", "cv7", "cv10"])
def test_table2_layers_small_batch(cuda_ok, name, dtype):
    """Every Table 2 layer shape at batch 2: spans many tiles, ragged M tails,
    Kdim tails (363, 147, 27), k_c = 512 (two N tiles), i_c = 3 lowering."""
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (2, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=2000 + int(name[2:]))
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    O_auto, g_auto = mec.conv_forward(Id, Kd, s, s, return_gemm=True)
    other = (MEC_PATH_SOLUTION_B if mec.select_path(shape, s, s) == MEC_PATH_SOLUTION_A
             else MEC_PATH_SOLUTION_A)
    O_other, g_other = mec.conv_forward(Id, Kd, s, s, path=other, return_gemm=True)
    torch.cuda.synchronize()
    check_O(O_auto, ref, dtype, k_h * k_w * i_c)
    check_O(O_other, ref, dtype, k_h * k_w * i_c)
    if 3 not in (g_auto, g_other):  # same MMA sequence per element unless split-K regrouped it
        assert torch.equal(O_auto, O_other)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_full24_values_within_north_star_tolerance(cuda_ok, dtype):
    # realistic (non-grid) fp32 values: tf32 / bf16 input rounding is now part of the error
    shape, s = (2, 56, 56, 64, 3, 3, 64), 1
    I, K = make_inputs(shape, "tf32", seed=5, kind=synth.KIND_FULL24)
    ref_vals_I = I if dtype == "tf32" else torch.from_numpy(I).to(torch.bfloat16).float().numpy()
    ref_vals_K = K if dtype == "tf32" else torch.from_numpy(K).to(torch.bfloat16).float().numpy()
    ref = oracle.direct_conv(ref_vals_I, ref_vals_K, s, s, n_threads=8)
    O = mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s)
    check_O(O, ref, dtype, 576, tight=False)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("rpt", [2, 3, 4, 8])
@pytest.mark.parametrize("name,batch", [("cv9", 3), ("cv10", 2), ("cv11", 2), ("cv8", 1)])
def test_multi_row_tiles(cuda_ok, name, batch, rpt, dtype):
    """Multi-row schedule (rows_per_tile): each streamed window atom feeds the
    MMAs of up to R output rows; must equal the one-row schedule bit for bit
    (same per-accumulator MMA order) and the oracle within tolerance."""
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=3000 + rpt)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    for path in (MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B):
        # (the one-row schedule of the same kernel: the automatic choice may be
        # the CTA-pair kernel, whose split-K regroups the sums)
        O1 = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=1)
        OR = mec.conv_forward(Id, Kd, s, s, path=path, rows_per_tile=rpt)
        torch.cuda.synchronize()
        check_O(OR, ref, dtype, k_h * k_w * i_c)
        assert torch.equal(O1, OR)


FUSED_CASES = [("cv4", 1), ("cv6", 3), ("cv8", 1), ("cv9", 3), ("cv10", 2), ("cv11", 3), ("cv12", 5)]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("name,batch", FUSED_CASES)
def test_fused_path(cuda_ok, name, batch, dtype):
    """MEC_PATH_FUSED (section 8 row a6): K-atoms of each window read as TMA boxes of
    I, L never written.  Same MMA sequence as the two-kernel path -> bit-identical."""
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=4000 + int(name[2:]))
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    OF, chosen = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_FUSED, return_path=True)
    O2 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_B)
    torch.cuda.synchronize()
    assert chosen == MEC_PATH_FUSED
    check_O(OF, ref, dtype, k_h * k_w * i_c)
    assert torch.equal(OF, O2)


# (layer, batch, dtype, the path MEC_PATH_FASTEST resolves to): the fused h-sweep on the
# HBM-bound wide-channel layers; the paper's Alg.2 l.8 choice on the tensor-bound ones,
# the 3-channel ones (no TMA-box fused variant) and tf32 VGG conv1_2 (window past the ring)
FASTEST_CASES = [("vgg16_conv1_2", 2, "bf16", "fused"), ("cv9", 3, "bf16", "fused"), ("cv8", 1, "bf16", "fused"),
                 ("cv12", 5, "bf16", "paper"), ("cv3", 2, "bf16", "paper"), ("vgg16_conv1_2", 1, "tf32", "paper")]


@pytest.mark.parametrize("name,batch,dtype,want", FASTEST_CASES)
def test_fastest_path(cuda_ok, name, batch, dtype, want):
    """MEC_PATH_FASTEST: the fused path where its TMA-box h-sweep applies and the
    layer is not tensor-bound, else MEC_PATH_AUTO's Alg.2 l.8 choice; either way
    within tolerance of the oracle and equal to the explicitly requested path."""
    from paper_1706_06873_b200._lib import MEC_PATH_AUTO, MEC_PATH_FASTEST, MEC_PATH_FUSED
    if name == "vgg16_conv1_2":
        i_h, i_w, i_c, k_h, k_w, k_c, s = 226, 226, 64, 3, 3, 64, 1
    else:
        i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=4300 + batch + len(name))
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    O, chosen = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_FASTEST, return_path=True)
    paper = mec.select_path(shape, s, s)
    assert chosen == (MEC_PATH_FUSED if want == "fused" else paper)
    O2 = mec.conv_forward(Id, Kd, s, s, path=chosen)
    torch.cuda.synchronize()
    check_O(O, ref, dtype, k_h * k_w * i_c)
    assert torch.equal(O, O2)
    if want == "paper":
        O3 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_AUTO)
        torch.cuda.synchronize()
        assert torch.equal(O, O3)


@pytest.mark.parametrize("shape,s", [((4, 56, 56, 256, 1, 1, 64), 1), ((3, 28, 28, 192, 1, 1, 64), 1),
                                     ((2, 30, 33, 64, 3, 3, 96), 2), ((2, 17, 140, 128, 2, 3, 48), 1)])
def test_fused_path_misc(cuda_ok, shape, s):
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    I, K = make_inputs(shape, "bf16", seed=77)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    OF = mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, path=MEC_PATH_FUSED)
    check_O(OF, ref, "bf16", shape[3] * shape[4] * shape[5])


GATHER_CASES = [("cv1", 3), ("cv2", 2), ("cv3", 2), ("cv7", 1)]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("name,batch", GATHER_CASES)
def test_fused_gather_path(cuda_ok, name, batch, dtype):
    """MEC_PATH_FUSED for small i_c (AlexNet conv1 and co.): input rows staged by
    bulk copies, A rows assembled in tensor memory by builder warps, L never written."""
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=5000 + int(name[2:]))
    if dtype == "tf32" and name in ("cv1", "cv2"):
        # fp32 weights of an 11x11x3x96 kernel (147 KB) cannot stay resident next to
        # the staged rows: the fused gather path refuses, the two-kernel path runs it
        with pytest.raises(MecError):
            mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s, path=MEC_PATH_FUSED)
        return
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    OF, chosen = mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s, path=MEC_PATH_FUSED,
                                  return_path=True)
    torch.cuda.synchronize()
    assert chosen == MEC_PATH_FUSED
    check_O(OF, ref, dtype, k_h * k_w * i_c)


@pytest.mark.parametrize("shape,s", [((3, 9, 11, 3, 3, 5, 8), 1), ((2, 30, 16, 64, 3, 3, 32), 3),
                                     ((5, 23, 21, 6, 3, 3, 24), 2), ((2, 40, 38, 5, 4, 3, 40), 1)])
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_fused_gather_misc(cuda_ok, shape, s, dtype):
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    I, K = make_inputs(shape, dtype, seed=91)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    OF = mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s, path=MEC_PATH_FUSED)
    check_O(OF, ref, dtype, shape[3] * shape[4] * shape[5])


def test_fused_gather_C1_full_batch_sampled(cuda_ok):
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    sampled_parity("C1", "bf16", [0, 13, 31], path=MEC_PATH_FUSED)


def test_fused_path_unsupported_shapes(cuda_ok):
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    I = torch.zeros(1, 20, 20, 3, device="cuda", dtype=torch.bfloat16)
    K = torch.zeros(3, 3, 3, 300, device="cuda", dtype=torch.bfloat16)  # two N tiles: not fused
    with pytest.raises(MecError):
        mec.conv_forward(I, K, 1, 1, path=MEC_PATH_FUSED)


# ------------------------------------------------------------------ lowering

LOWER_CASES = [
    ((2, 227, 227, 3, 11, 11, 1), 4, 4),   # cv1: 66-byte strips, unaligned segments
    ((3, 56, 56, 64, 3, 3, 1), 1, 1),      # cv9: aligned fast path
    ((2, 231, 231, 3, 11, 11, 1), 4, 4),   # cv2
    ((2, 224, 224, 64, 7, 7, 1), 2, 2),    # cv4: unused last input row (Q5)
    ((1, 7, 7, 1, 3, 3, 1), 1, 1),         # C0
    ((2, 12, 12, 7, 2, 2, 1), 3, 3),       # s > k
    ((2, 13, 9, 5, 1, 1, 1), 1, 1),        # 1x1
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(LOWER_CASES)))
def test_lowering_bit_exact(cuda_ok, case, dtype):
    shape, s_h, s_w = LOWER_CASES[case]
    i_n, i_h, i_w, i_c, k_h, k_w, _ = shape
    # arbitrary bit patterns (incl. NaN/Inf encodings): the lowering is a pure copy
    rng = np.random.default_rng(case)
    if dtype == "bf16":
        bits = rng.integers(0, 2**16, (i_n, i_h, i_w, i_c), dtype=np.uint16)
        Id = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        bits = rng.integers(0, 2**32, (i_n, i_h, i_w, i_c), dtype=np.uint32)
        Id = torch.from_numpy(bits.view(np.int32)).cuda().view(torch.float32)
    L = mec.lower(Id, k_h, k_w, s_h, s_w)
    ref = oracle.lower(bits, k_h, k_w, s_h, s_w)
    got = L.cpu().view(torch.int16 if dtype == "bf16" else torch.int32).numpy()
    np.testing.assert_array_equal(got.view(ref.dtype), ref)


PITCHED_CASES = LOWER_CASES + [
    ((2, 227, 227, 3, 7, 7, 1), 2, 2),     # cv3: 42-byte strips, 4 alignment classes
    ((2, 224, 224, 3, 3, 3, 1), 1, 1),     # cv7: 18-byte strips, 8 classes (word-table path)
    ((3, 40, 37, 3, 5, 4, 1), 3, 2),       # odd extents, ragged last band
    ((1, 19, 23, 5, 4, 3, 1), 2, 1),       # 30-byte strips, i_c = 5
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(PITCHED_CASES)))
def test_lowering_pitched_bit_exact(cuda_ok, case, dtype):
    """The conv path's pitch-padded L (mec_lower_pitched, the layout the window
    GEMM reads) holds exactly the oracle's lowering in every row's first
    i_h k_w i_c elements, for the default 16-byte pitch and a wider one."""
    shape, s_h, s_w = PITCHED_CASES[case]
    i_n, i_h, i_w, i_c, k_h, k_w, _ = shape
    rng = np.random.default_rng(100 + case)
    if dtype == "bf16":
        bits = rng.integers(0, 2**16, (i_n, i_h, i_w, i_c), dtype=np.uint16)
        Id = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        bits = rng.integers(0, 2**32, (i_n, i_h, i_w, i_c), dtype=np.uint32)
        Id = torch.from_numpy(bits.view(np.int32)).cuda().view(torch.float32)
    ref = oracle.lower(bits, k_h, k_w, s_h, s_w)
    cols = i_h * k_w * i_c
    ref = ref.reshape(-1, cols)
    v = 16 // Id.element_size()
    for pitch in ((cols + v - 1) // v * v, (cols + v - 1) // v * v + 3 * v):
        Lp = mec.lower_pitched(Id, k_h, k_w, s_h, s_w, pitch=pitch)
        got = Lp.cpu().view(torch.int16 if dtype == "bf16" else torch.int32).numpy()[:, :cols]
        np.testing.assert_array_equal(got.view(ref.dtype), ref)


def test_lowering_pitched_full_C1_bit_exact(cuda_ok):
    c = synth.config("C1")
    I, _ = make_inputs((c["i_n"], c["i_h"], c["i_w"], c["i_c"], c["k_h"], c["k_w"], c["k_c"]), "bf16", seed=2)
    Id = to_dev(I, "bf16")
    Lp = mec.lower_pitched(Id, c["k_h"], c["k_w"], c["s_h"], c["s_w"])
    bits = Id.view(torch.int16).cpu().numpy()
    ref = oracle.lower(bits, c["k_h"], c["k_w"], c["s_h"], c["s_w"])
    cols = c["i_h"] * c["k_w"] * c["i_c"]
    np.testing.assert_array_equal(Lp.view(torch.int16).cpu().numpy()[:, :cols], ref.reshape(-1, cols))


def test_lowering_full_C1_batch_bit_exact(cuda_ok):
    c = synth.config("C1")
    I, _ = make_inputs((c["i_n"], c["i_h"], c["i_w"], c["i_c"], c["k_h"], c["k_w"], c["k_c"]), "bf16", seed=1)
    Id = to_dev(I, "bf16")
    L = mec.lower(Id, c["k_h"], c["k_w"], c["s_h"], c["s_w"])
    bits = Id.view(torch.int16).cpu().numpy()
    ref = oracle.lower(bits, c["k_h"], c["k_w"], c["s_h"], c["s_w"])
    np.testing.assert_array_equal(L.view(torch.int16).cpu().numpy(), ref)


# -------------------------------------------- BASELINE configs at full size

def sampled_parity(cfg_name, dtype, images, path=0, batch=None):
    """The whole batch at the bench's size (bench.py's launch configuration:
    inputs generated on the device, one mec_conv_forward_ex call on the full
    batch), then the sampled images recomputed by the oracle one by one."""
    c = synth.config(cfg_name, batch)
    shape = (c["i_n"], c["i_h"], c["i_w"], c["i_c"], c["k_h"], c["k_w"], c["k_c"])
    seed = synth.SEED_BASE + c["index"]
    kind = synth.KIND_GRID8 if dtype == "bf16" else synth.KIND_GRID11
    # the full batch generated on the device (bench's launch configuration) ...
    Id = torch.empty(shape[:4], dtype=TDT[dtype], device="cuda")
    Kd = torch.empty((c["k_h"], c["k_w"], c["i_c"], c["k_c"]), dtype=TDT[dtype], device="cuda")
    mec.synth_fill(Id, seed, synth.TENSOR_I, kind)
    mec.synth_fill(Kd, seed, synth.TENSOR_K, kind)
    O = mec.conv_forward(Id, Kd, c["s_h"], c["s_w"], path=path)
    torch.cuda.synchronize()
    del Id
    # ... and the sampled images regenerated on the host for the oracle
    K = synth.kernel_tensor(c, kind, seed)
    np.testing.assert_array_equal(Kd.float().cpu().numpy(), K)
    for n in images:
        n = n % c["i_n"]
        I = synth.input_images(c, n, 1, kind, seed)
        ref = oracle.direct_conv(I, K, c["s_h"], c["s_w"], n_threads=8)
        check_O(O[n:n + 1], ref, dtype, c["k_h"] * c["k_w"] * c["i_c"])
    del O
    torch.cuda.empty_cache()


C4_LAYERS = list(synth.TABLE2) + list(synth.ONE_BY_ONE)


@pytest.mark.parametrize("layer", C4_LAYERS)
def test_C4_sweep_b128_sampled(cuda_ok, layer):
    """C4 at b128 (the per-GPU shard of b1024 at g = 8, the size bench.py times
    for the sweep lines): the first, a middle and the last image."""
    sampled_parity(f"C4_{layer}", "bf16", [0, 77, -1], batch=128)


@pytest.mark.parametrize("layer", ["cv4", "cv5", "cv12"])
def test_C4_sweep_b1024_sampled(cuda_ok, layer):
    """C4 at its stated batch 1024 (cv4: a 22.4 GB L, index math past 2^32 bytes)."""
    sampled_parity(f"C4_{layer}", "bf16", [0, 513, -1], batch=1024)


@pytest.mark.parametrize("layer", ["cv4", "cv5"])
def test_C4_tf32_b128_sampled(cuda_ok, layer):
    """C4's tf32 rows (+tf32 on cv4, cv5)."""
    c = synth.config(f"C4_{layer}", 128)
    synth.CONFIGS[f"_tmp_{layer}_tf32"] = dict(c, dtype="tf32")
    try:
        sampled_parity(f"_tmp_{layer}_tf32", "tf32", [0, -1])
    finally:
        del synth.CONFIGS[f"_tmp_{layer}_tf32"]


def test_C1_alexnet_conv1_full_batch_sampled(cuda_ok):
    sampled_parity("C1", "bf16", [0, 17, 31])


@pytest.mark.parametrize("path", [MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B])
def test_C3_resnet50_stage2_full_batch_sampled(cuda_ok, path):
    sampled_parity("C3", "bf16", [0, 128, 255], path=path)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_C2_vgg_conv1_2_full_batch_sampled(cuda_ok, dtype):
    sampled_parity("C2" if dtype == "bf16" else "C2_tf32", dtype, [0, 63])


# ------------------------------------------------------------- generator

@pytest.mark.parametrize("kind", [synth.KIND_GRID8, synth.KIND_GRID11, synth.KIND_FULL24])
def test_device_generator_matches_host(cuda_ok, kind):
    t = torch.empty(100003, dtype=torch.float32, device="cuda")
    mec.synth_fill(t, 12345, 1, kind, index_offset=777)
    np.testing.assert_array_equal(t.cpu().numpy(), synth.draw(100003, 12345, 1, kind, 777))
    if kind == synth.KIND_GRID8:
        tb = torch.empty(1000, dtype=torch.bfloat16, device="cuda")
        mec.synth_fill(tb, 12345, 1, kind, index_offset=777)
        np.testing.assert_array_equal(tb.float().cpu().numpy(), synth.draw(1000, 12345, 1, kind, 777))


# ---------------------------------------------------------------- errors

def test_error_paths_on_device(cuda_ok):
    I = torch.zeros(1, 7, 7, 1, device="cuda")
    K = torch.zeros(3, 3, 1, 1, device="cuda")
    with pytest.raises(MecError):  # misaligned I
        mec.conv_forward(torch.zeros(50, device="cuda")[1:50].view(1, 7, 7, 1), K, 1, 1)
    with pytest.raises(MecError):  # i < k
        mec.conv_forward(torch.zeros(1, 2, 7, 1, device="cuda"), K, 1, 1)
    ws = torch.empty(mec.workspace_bytes((1, 7, 7, 1, 3, 3, 1), 1, 1, torch.float32), dtype=torch.uint8,
                     device="cuda")
    O = mec.conv_forward(I, K, 1, 1, workspace=ws)
    assert float(O.abs().max()) == 0.0
    with pytest.raises(MecError):
        mec.conv_forward(I, K, 1, 1, workspace=ws[: ws.numel() // 2])


# ------------------------------------------------ NEXT-2: stride sweep on cv1

_STRIDE_REF = {}


def _stride_case(s):
    """cv1 geometry (Table 2: 227x227x3, 11x11, k_c 96) at stride s (Fig. 4(a))."""
    i_h, i_w, i_c, k_h, k_w, k_c, _ = synth.TABLE2["cv1"]
    shape = (1, i_h, i_w, i_c, k_h, k_w, k_c)
    if s not in _STRIDE_REF:
        I, K = make_inputs(shape, "bf16", seed=7000 + s)
        _STRIDE_REF[s] = (I, K, oracle.direct_conv(I, K, s, s, n_threads=8))
    return shape, _STRIDE_REF[s]


@pytest.mark.parametrize("path", ["auto", "fused"])
@pytest.mark.parametrize("s", range(1, 11))
def test_cv1_stride_sweep(cuda_ok, s, path):
    """s = 1..10 exercises s >= k/2, strides that do not divide i - k, and input rows
    no GEMM reads (reading Q5); the AUTO path follows Alg.2 l.8 at every s."""
    from paper_1706_06873_b200._lib import MEC_PATH_AUTO, MEC_PATH_FUSED
    shape, (I, K, ref) = _stride_case(s)
    p = MEC_PATH_FUSED if path == "fused" else MEC_PATH_AUTO
    O, chosen = mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, path=p, return_path=True)
    torch.cuda.synchronize()
    if path == "auto":
        assert chosen == oracle.select_path(shape, s, s, 100)
    check_O(O, ref, "bf16", shape[3] * shape[4] * shape[5])


# ------------------------------------- NEXT-4: zero padding inside the lowering
# P:41 assumes I already zero-padded.  The library pads virtually; the reference
# is the oracle on the explicitly padded array (np.pad: a host-side data step,
# not oracle arithmetic).

PAD_LOWER_CASES = [
    # shape, s_h, s_w, pad_h, pad_w
    ((2, 9, 11, 3, 3, 3, 1), 1, 1, 1, 1),      # i_c = 3, general (word-table) path
    ((2, 14, 14, 64, 3, 3, 1), 1, 1, 1, 1),    # aligned (128-bit) path
    ((1, 20, 17, 3, 7, 7, 1), 2, 2, 3, 3),     # ResNet conv1-like, stride 2
    ((2, 12, 10, 5, 5, 3, 1), 2, 1, 2, 0),     # asymmetric pads
    ((1, 7, 7, 1, 3, 3, 1), 1, 1, 0, 2),       # width padding only
]


def _pad(a, ph, pw):
    return np.pad(a, ((0, 0), (ph, ph), (pw, pw), (0, 0)))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(PAD_LOWER_CASES)))
def test_padded_lowering_bit_exact(cuda_ok, case, dtype):
    shape, s_h, s_w, ph, pw = PAD_LOWER_CASES[case]
    i_n, i_h, i_w, i_c, k_h, k_w, _ = shape
    rng = np.random.default_rng(100 + case)
    if dtype == "bf16":
        bits = rng.integers(0, 2**16, (i_n, i_h, i_w, i_c), dtype=np.uint16)
        Id = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        bits = rng.integers(0, 2**32, (i_n, i_h, i_w, i_c), dtype=np.uint32)
        Id = torch.from_numpy(bits.view(np.int32)).cuda().view(torch.float32)
    L = mec.lower(Id, k_h, k_w, s_h, s_w, pad_h=ph, pad_w=pw)
    ref = oracle.lower(_pad(bits, ph, pw), k_h, k_w, s_h, s_w)
    got = L.cpu().view(torch.int16 if dtype == "bf16" else torch.int32).numpy()
    np.testing.assert_array_equal(got.view(ref.dtype), ref)


PAD_CONV_CASES = [
    # shape, s, pad_h, pad_w
    ((2, 14, 14, 64, 3, 3, 64), 1, 1, 1),      # ResNet 3x3 "same"
    ((2, 32, 32, 3, 7, 7, 64), 2, 3, 3),       # ResNet conv1 geometry (reduced)
    ((3, 11, 13, 8, 5, 3, 24), 2, 2, 1),       # asymmetric, k_c not a multiple of 16
    ((2, 9, 9, 128, 3, 3, 32), 2, 1, 1),       # fused TMA variant eligible (i_c elt = 256 B)
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("path", ["A", "B", "fused"])
@pytest.mark.parametrize("case", range(len(PAD_CONV_CASES)))
def test_padded_conv(cuda_ok, case, path, dtype):
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    shape, s, ph, pw = PAD_CONV_CASES[case]
    I, K = make_inputs(shape, dtype, seed=300 + case)
    ref = oracle.direct_conv(_pad(I, ph, pw), K, s, s, n_threads=8)
    p = {"A": MEC_PATH_SOLUTION_A, "B": MEC_PATH_SOLUTION_B, "fused": MEC_PATH_FUSED}[path]
    i_c = shape[3]
    if path == "fused" and (i_c * (2 if dtype == "bf16" else 4)) % 128 != 0:
        # the gather variant copies staged rows verbatim: padded problems are refused
        with pytest.raises(MecError):
            mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s, path=p, pad_h=ph, pad_w=pw)
        return
    O = mec.conv_forward(to_dev(I, dtype), to_dev(K, dtype), s, s, path=p, pad_h=ph, pad_w=pw)
    torch.cuda.synchronize()
    check_O(O, ref, dtype, shape[3] * shape[4] * shape[5])


# --------------------- NEXT-4: pooling consumes Solution A's h-n-w-c

def _maxpool_ref(X, p_h, p_w, s_h, s_w):
    """Definition: Y[n,y,x,c] = max over the p_h x p_w window at (y s_h, x s_w)."""
    from numpy.lib.stride_tricks import sliding_window_view
    win = sliding_window_view(X, (p_h, p_w), axis=(1, 2))[:, ::s_h, ::s_w]
    return win.max(axis=(-2, -1))


POOL_CASES = [
    # conv shape, conv stride, (pool window, pool stride)
    ((2, 35, 35, 3, 11, 11, 96), 4, (3, 2)),   # AlexNet conv1 -> pool1 geometry (reduced)
    ((3, 20, 20, 16, 3, 3, 64), 1, (2, 2)),
    ((2, 16, 19, 8, 3, 3, 32), 1, (3, 3)),
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(POOL_CASES)))
def test_maxpool_consumes_hnwc(cuda_ok, case, dtype):
    shape, s, (pk, ps) = POOL_CASES[case]
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
    I, K = make_inputs(shape, dtype, seed=400 + case)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    O_nhwc = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, sola_fix=MEC_SOLA_FIX_EPILOGUE)
    O_raw = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, sola_fix=MEC_SOLA_FIX_NONE)
    o_h, o_w = O_nhwc.shape[1], O_nhwc.shape[2]
    O_hnwc = O_raw.view(o_h, i_n, o_w, k_c)  # Alg.2 l.10: O as o_h x i_n o_w k_c
    assert torch.equal(O_hnwc.permute(1, 0, 2, 3), O_nhwc)
    Y_h = mec.maxpool(O_hnwc, pk, pk, ps, ps, hnwc=True)
    Y_n = mec.maxpool(O_nhwc, pk, pk, ps, ps)
    torch.cuda.synchronize()
    assert torch.equal(Y_h, Y_n)  # the transpose was never needed
    np.testing.assert_array_equal(Y_n.float().cpu().numpy(),
                                  _maxpool_ref(O_nhwc.float().cpu().numpy(), pk, pk, ps, ps))
    ref = _maxpool_ref(oracle.direct_conv(I, K, s, s, n_threads=8), pk, pk, ps, ps)
    check_O(Y_n, ref, dtype, i_c * k_h * k_w)


# The h-sweep window GEMM against the oracle and against the
# one-window-per-tile kernel: shapes with 1, 2, 4 and 8 shifted weight variants,
# one and two MMA issuers, packed / flat (o_w < 32) Solution A tiles and
# Solution B with two M tiles per image (o_w > 128).
SWEEP_CASES = [
    ((2, 227, 227, 3, 11, 11, 96), 4),   # AlexNet conv1: 2 variants, 1 issuer
    ((2, 224, 224, 3, 7, 7, 64), 2),     # cv3: 4 variants
    ((2, 64, 64, 3, 3, 3, 64), 1),       # cv7-like: 8 variants, many rows per atom
    ((3, 56, 56, 64, 3, 3, 64), 1),      # cv9: 1 variant, 2 issuers
    ((4, 20, 20, 64, 3, 3, 64), 1),      # o_w = 18: flat Solution A tiles
    ((2, 140, 140, 64, 3, 3, 64), 1),    # o_w = 138: two M tiles per image
    ((2, 30, 30, 32, 5, 5, 48), 2),      # k_c = 48, stride 2
    ((2, 30, 30, 64, 3, 3, 128), 1),     # k_c = 128: one TMEM accumulator
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(SWEEP_CASES)))
def test_sweep_gemm_vs_oracle_and_one_window(cuda_ok, case, dtype):
    shape, s = SWEEP_CASES[case]
    I, K = make_inputs(shape, dtype, seed=6100 + case)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    kdim = shape[4] * shape[5] * shape[3]
    outs = {}
    for path in (MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B):
        try:
            O, g = mec.conv_forward(Id, Kd, s, s, path=path, return_gemm=True)
        except MecError:  # (Solution A infeasible when #O > #L)
            continue
        O1, g1 = mec.conv_forward(Id, Kd, s, s, path=path, rows_per_tile=1, return_gemm=True)
        torch.cuda.synchronize()
        assert g1 == 1
        check_O(O, ref, dtype, kdim)
        check_O(O1, ref, dtype, kdim)
        outs[path] = (O, g)
    assert outs, "no path ran"
    gs = {g for _, g in outs.values()}
    # Solutions A and B may pick different window-GEMM kernels (each checked
    # against the oracle above); with one kernel for both, or the one-window
    # kernel and the pair sweep (the same K steps per row), they agree bitwise
    if len(outs) == 2 and (len(gs) == 1 or gs <= {1, 4}):  # Solutions A and B: the same K steps per row -> bitwise equal (reading Q10)
        assert torch.equal(outs[MEC_PATH_SOLUTION_A][0], outs[MEC_PATH_SOLUTION_B][0])


def test_sweep_gemm_selected_for_C1_C2_C3(cuda_ok):
    """The configs the bench times run the h-sweep kernel (bf16)."""
    for shape, s in [((1, 227, 227, 3, 11, 11, 96), 4), ((1, 224, 224, 64, 3, 3, 64), 1),
                     ((2, 56, 56, 64, 3, 3, 64), 1)]:
        I, K = make_inputs(shape, "bf16", seed=6200)
        _, g = mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, return_gemm=True)
        assert g == 2, shape


# ---- end to end on host buffers (mec_conv_forward_host): copies pipelined over image chunks
HOST_CASES = [
    # shape, s_h, s_w, n_chunks (ragged last chunk, more chunks than slots, chunks > i_n clamped)
    ((5, 20, 17, 5, 4, 3, 24), 2, 1, 2),
    ((7, 30, 30, 16, 3, 3, 40), 1, 1, 4),
    ((3, 12, 12, 7, 2, 2, 17), 3, 3, 9),
    ((6, 27, 27, 3, 11, 11, 96), 4, 4, 6),
    ((1, 8, 9, 6, 8, 9, 48), 1, 1, 1),
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(HOST_CASES)))
def test_conv_forward_host_pipelined(cuda_ok, case, dtype):
    """The host-buffer call equals the oracle, and equals the device call element for element
    (each chunk is a sub-batch of the same Algorithm 2 path: the arithmetic per output element
    does not depend on the chunking)."""
    shape, s_h, s_w, nch = HOST_CASES[case]
    I, K = make_inputs(shape, dtype, seed=7000 + case)
    ref = oracle.direct_conv(I, K, s_h, s_w)
    I_h = torch.from_numpy(np.ascontiguousarray(I)).to(TDT[dtype]).pin_memory()
    K_h = torch.from_numpy(np.ascontiguousarray(K)).to(TDT[dtype]).pin_memory()
    O_h, path = mec.conv_forward_host(I_h, K_h, s_h, s_w, n_chunks=nch, return_path=True)
    torch.cuda.synchronize()
    assert path == mec.select_path(shape, s_h, s_w)
    check_O(O_h, ref, dtype, shape[4] * shape[5] * shape[3])
    O_d = mec.conv_forward(I_h.cuda(), K_h.cuda(), s_h, s_w)
    torch.cuda.synchronize()
    assert torch.equal(O_h, O_d.cpu())


def test_conv_forward_host_scratch_and_repeat(cuda_ok):
    """Caller scratch, pageable host memory, back-to-back calls reusing the library's streams
    and events, and a too-small scratch (MEC_ERR_NO_MEMORY)."""
    shape, s = (9, 27, 27, 3, 11, 11, 96), 4
    I, K = make_inputs(shape, "bf16", seed=7100)
    ref = oracle.direct_conv(I, K, s, s)
    I_h = torch.from_numpy(I).to(torch.bfloat16)  # pageable
    K_h = torch.from_numpy(K).to(torch.bfloat16)
    nb = mec.host_scratch_bytes(*shape, s, s, torch.bfloat16, 4)
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda")
    outs = [mec.conv_forward_host(I_h, K_h, s, s, n_chunks=4, scratch=scratch) for _ in range(3)]
    torch.cuda.synchronize()
    for O in outs:
        check_O(O, ref, "bf16", 11 * 11 * 3)
        assert torch.equal(O, outs[0])
    with pytest.raises(MecError):
        mec.conv_forward_host(I_h, K_h, s, s, n_chunks=4, scratch=scratch[:nb - 2048])
    with pytest.raises(MecError):
        mec.conv_forward_host(I_h, K_h, s, s, sola_fix=MEC_SOLA_FIX_NONE)


def test_C1_conv_forward_host_full_batch_sampled(cuda_ok):
    """The bench's e2e launch configuration: C1 at its full batch through the host-buffer call."""
    c = synth.config("C1")
    shape = (c["i_n"], c["i_h"], c["i_w"], c["i_c"], c["k_h"], c["k_w"], c["k_c"])
    seed = synth.SEED_BASE + c["index"]
    kind = synth.KIND_GRID8
    Id = torch.empty(shape[:4], dtype=torch.bfloat16, device="cuda")
    Kd = torch.empty((c["k_h"], c["k_w"], c["i_c"], c["k_c"]), dtype=torch.bfloat16, device="cuda")
    mec.synth_fill(Id, seed, synth.TENSOR_I, kind)
    mec.synth_fill(Kd, seed, synth.TENSOR_K, kind)
    I_h, K_h = Id.cpu().pin_memory(), Kd.cpu().pin_memory()
    O = mec.conv_forward_host(I_h, K_h, c["s_h"], c["s_w"], n_chunks=4)
    torch.cuda.synchronize()
    K = synth.kernel_tensor(c, kind, seed)
    for n in [0, 13, 31]:
        I = synth.input_images(c, n, 1, kind, seed)
        ref = oracle.direct_conv(I, K, c["s_h"], c["s_w"], n_threads=8)
        check_O(O[n:n + 1], ref, "bf16", c["k_h"] * c["k_w"] * c["i_c"])


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("path", ["A", "B", "fused"])
def test_conv_forward_host_padded_and_forced_paths(cuda_ok, path, dtype):
    """The host-buffer call with virtual zero padding and each forced path (the fused TMA variant
    included), over chunks with a ragged tail: equal to the oracle on the padded input."""
    from paper_1706_06873_b200._lib import MEC_PATH_FUSED
    shape, s, ph, pw = (5, 9, 9, 128, 3, 3, 32), 2, 1, 1
    I, K = make_inputs(shape, dtype, seed=7200)
    ref = oracle.direct_conv(_pad(I, ph, pw), K, s, s, n_threads=8)
    p = {"A": MEC_PATH_SOLUTION_A, "B": MEC_PATH_SOLUTION_B, "fused": MEC_PATH_FUSED}[path]
    I_h = torch.from_numpy(np.ascontiguousarray(I)).to(TDT[dtype]).pin_memory()
    K_h = torch.from_numpy(np.ascontiguousarray(K)).to(TDT[dtype]).pin_memory()
    O, ran = mec.conv_forward_host(I_h, K_h, s, s, n_chunks=3, path=p, pad_h=ph, pad_w=pw, return_path=True)
    torch.cuda.synchronize()
    assert ran == p
    check_O(O, ref, dtype, shape[3] * shape[4] * shape[5])


# ------------------------------------------- the C ABI's named entry points

def test_abi_named_calls_conv_forward_and_lower(cuda_ok):
    """north_star's two named calls, mec_conv_forward and mec_lower, called by
    name through ctypes (not the _ex / _padded variants the binding uses)."""
    import ctypes

    from paper_1706_06873_b200 import _lib

    L_ = _lib.lib()
    shape, s = (3, 19, 23, 16, 3, 3, 32), 2
    I, K = make_inputs(shape, "bf16", seed=4242)
    Id, Kd = to_dev(I, "bf16"), to_dev(K, "bf16")
    ref = oracle.direct_conv(I, K, s, s)
    O = torch.empty(ref.shape, dtype=torch.bfloat16, device="cuda")
    sh = _lib.MecShape(*shape)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L_.mec_conv_forward(Id.data_ptr(), Kd.data_ptr(), O.data_ptr(), ctypes.byref(sh), s, s,
                               _lib.MEC_DTYPE_BF16, stream) == 0
    torch.cuda.synchronize()
    check_O(O, ref, "bf16", 3 * 3 * 16)
    o_w = (23 - 3) // s + 1
    Ld = torch.empty((3, o_w, 19, 3, 16), dtype=torch.bfloat16, device="cuda")
    assert L_.mec_lower(Id.data_ptr(), Ld.data_ptr(), ctypes.byref(sh), s, s, _lib.MEC_DTYPE_BF16, stream) == 0
    torch.cuda.synchronize()
    bits = Id.view(torch.int16).cpu().numpy()
    np.testing.assert_array_equal(Ld.view(torch.int16).cpu().numpy(), oracle.lower(bits, 3, 3, s, s))


@pytest.mark.parametrize("path", [MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B])
def test_non_finite_input_documented_behaviour(cuda_ok, path):
    """include/mec.h: inputs must be finite.  Pinned behaviour with one NaN
    pixel in I: every output whose window holds it (the definition) is
    NaN; the K-tail of a window box may also reach it from a neighbouring
    window (zero weights times NaN), so further outputs MAY be NaN; every
    output that is finite equals the oracle within the tolerance."""
    shape, s = (2, 12, 13, 8, 3, 3, 16), 1
    I, K = make_inputs(shape, "tf32", seed=99)
    I[1, 5, 6, 3] = np.nan
    ref = oracle.direct_conv(I, K, s, s)
    O = mec.conv_forward(to_dev(I, "tf32"), to_dev(K, "tf32"), s, s, path=path)
    torch.cuda.synchronize()
    got = O.cpu().numpy().astype(np.float64)
    nan_ref, nan_got = np.isnan(ref), np.isnan(got)
    assert nan_ref.sum() == 3 * 3 * 16  # the 3x3 outputs (x 16 channels) whose windows hold the pixel
    assert np.all(nan_got[nan_ref])
    fin = ~nan_got
    bar = tol("tf32", 72, np.where(nan_ref, 0.0, ref))
    assert np.abs(got[fin] - ref[fin]).max() <= bar
    assert not np.any(nan_got[0])  # the other image is untouched


BAL_CASES = [
    # (name or shape, batch / stride, path)
    (("cv9", 8), MEC_PATH_SOLUTION_A),     # 4 tiles x 54 rows on 148 CTAs: 1-2 rows each, pieces across tiles
    (("cv1", 6), MEC_PATH_SOLUTION_A),     # AlexNet conv1 rows (2 weight variants), 3 tiles
    (("cv3", 3), MEC_PATH_SOLUTION_B),     # 7x7 s2, per-image tiles
    (((3, 30, 230, 64, 3, 3, 64), 1), MEC_PATH_SOLUTION_B),  # o_w 228: 2 CTA tiles per image
    (((3, 30, 230, 64, 3, 3, 64), 1), MEC_PATH_FUSED),       # the fused TMA-box variant
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(BAL_CASES)))
def test_sweep_balanced_split(cuda_ok, monkeypatch, case, dtype):
    """The h-sweep's balanced split (every CTA the same number of (tile, h) rows,
    cut at tile boundaries) against the chunked items: the same
    K steps per row, so bit for bit, and the oracle within tolerance."""
    (what, b), path = BAL_CASES[case]
    if isinstance(what, str):
        i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[what]
        shape = (b, i_h, i_w, i_c, k_h, k_w, k_c)
    else:
        shape, s = what, b
    if path == MEC_PATH_FUSED and dtype == "tf32":
        pytest.skip("fused TMA-box variant: bf16 case is enough here")
    I, K = make_inputs(shape, dtype, seed=6300 + case)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    outs = []
    for bal in ("1", "0"):
        monkeypatch.setenv("MEC_SWEEP_BALANCED", bal)
        try:
            O, g = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=2, return_gemm=True)
        except MecError:
            if dtype == "tf32":  # (a tf32 window wider than the TMEM ring: no h-sweep)
                pytest.skip("h-sweep does not apply to this tf32 window")
            raise
        torch.cuda.synchronize()
        assert g == 2
        outs.append(O)
    check_O(outs[0], ref, dtype, shape[4] * shape[5] * shape[3])
    assert torch.equal(outs[0], outs[1])


# ------------------------------- the CTA-pair (cta_group::2) split-K kernel

WIDE_CASES = [("cv12", 2), ("cv12", 9), ("cv6", 3), ("cv5", 2), ("cv11", 4), ("cv10", 3)]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("split", [0, 1, 2, 3, 5, 8])
@pytest.mark.parametrize("name,batch", WIDE_CASES)
def test_wide_pair_kernel(cuda_ok, name, batch, split, dtype):
    """Solution A on CTA pairs (M = 256 across two SMs) with K split
    into `split` ranges whose fp32 partials are summed in range order: within the
    north_star tolerance of the oracle, deterministic run to run, and with one
    range the same MMA sequence per element as the one-window kernel."""
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, dtype, seed=6000 + int(name[2:]) + batch)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    O, g, used = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=3, split_k=split,
                                  return_gemm=True, return_split=True)
    O2 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=3, split_k=split)
    torch.cuda.synchronize()
    assert g == 3 and used >= 1 and (split == 0 or used <= split)
    check_O(O, ref, dtype, k_h * k_w * i_c)
    assert torch.equal(O, O2)
    if used == 1:
        O1 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=1)
        torch.cuda.synchronize()
        assert torch.equal(O, O1)


@pytest.mark.parametrize("name,batch,forced", [("cv6", 128, None), ("cv11", 136, "1"), ("cv5", 48, "1")])
def test_wide_pair_kernel_hybrid_split(cuda_ok, monkeypatch, name, batch, forced):
    """Hybrid split: whole waves of unsplit pair tiles, then the
    last partial wave's tiles in S ranges that exchange partials (cv6 b128: 100
    tiles on 74 pairs, S = 2 by the cost model; cv11 b136: 84 tiles, S = 7 forced;
    cv5 b48: 80 tiles, S = 8 forced).  Sampled images against the oracle,
    deterministic run to run."""
    if forced is not None:
        monkeypatch.setenv("MEC_WIDE_HYBRID", forced)
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    seed = 6200 + batch
    Id = torch.empty(shape[:4], dtype=torch.bfloat16, device="cuda")
    Kd = torch.empty((k_h, k_w, i_c, k_c), dtype=torch.bfloat16, device="cuda")
    mec.synth_fill(Id, seed, synth.TENSOR_I, synth.KIND_GRID8)
    mec.synth_fill(Kd, seed, synth.TENSOR_K, synth.KIND_GRID8)
    O, g, used = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, return_gemm=True, return_split=True)
    O2 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A)
    torch.cuda.synchronize()
    assert g == 3 and used >= 2, (g, used)
    assert torch.equal(O, O2)
    cfg = dict(i_h=i_h, i_w=i_w, i_c=i_c, k_h=k_h, k_w=k_w, k_c=k_c)
    K = synth.kernel_tensor(cfg, synth.KIND_GRID8, seed)
    for n in (0, batch // 2, batch - 1):
        I = synth.input_images(cfg, n, 1, synth.KIND_GRID8, seed)
        ref = oracle.direct_conv(I, K, s, s, n_threads=8)
        check_O(O[n:n + 1], ref, "bf16", k_h * k_w * i_c)


def test_wide_pair_kernel_refuses_other_layouts(cuda_ok):
    """Forced CTA-pair kernel where it does not apply (per-image tiles of Solution B,
    k_c not a multiple of 32): MEC_ERR_UNSUPPORTED, not a silent fallback."""
    shape, s = (2, 30, 40, 64, 3, 3, 128), 1
    I, K = make_inputs(shape, "bf16", seed=1)
    with pytest.raises(MecError):
        mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, path=MEC_PATH_SOLUTION_B, gemm_kernel=3)
    shape = (2, 30, 40, 64, 3, 3, 40)
    I, K = make_inputs(shape, "bf16", seed=1)
    with pytest.raises(MecError):
        mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=3)


WIDE_WIDE_ROWS = [("cv1", 3), ("cv9", 5), ("cv2", 2)]


@pytest.mark.parametrize("split", [1, 2, 3])
@pytest.mark.parametrize("name,batch", WIDE_WIDE_ROWS)
def test_wide_pair_kernel_wide_rows(cuda_ok, name, batch, split):
    """The CTA-pair kernel on batch-folded rows of wider outputs (o_w >= 32: rows of
    several images share a 128-row half tile), with shifted weight copies (AlexNet
    conv1: window starts 264 bytes apart, 4 copies)."""
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, "bf16", seed=6100 + batch)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, "bf16"), to_dev(K, "bf16")
    O, g = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=3, split_k=split, return_gemm=True)
    torch.cuda.synchronize()
    assert g == 3
    check_O(O, ref, "bf16", k_h * k_w * i_c)
    if split == 1:
        O1 = mec.conv_forward(Id, Kd, s, s, path=MEC_PATH_SOLUTION_A, gemm_kernel=1)
        torch.cuda.synchronize()
        assert torch.equal(O, O1)


# ---------------------------- the CTA-pair atom-major sweep (gemm_kernel 4)

PS_CASES = [
    # shape, s, path
    ((3, 30, 230, 64, 3, 3, 64), 1, MEC_PATH_SOLUTION_B),   # VGG conv1_2-like rows (o_w 228: 2 CTA tiles per image)
    ((1, 20, 140, 64, 3, 3, 64), 1, MEC_PATH_SOLUTION_B),   # odd CTA-tile count: the last pair's second CTA is empty
    ((2, 40, 112, 64, 3, 3, 128), 1, MEC_PATH_SOLUTION_B),  # cv8-like (k_c 128: 4 accumulators)
    ((5, 56, 56, 64, 3, 3, 64), 1, MEC_PATH_SOLUTION_A),    # cv9 / C3 (2 image slots per CTA tile)
    ((3, 21, 80, 32, 5, 3, 48), 2, MEC_PATH_SOLUTION_A),    # s_h = 2, k_c 48, o_w 39 (64-row slots)
    ((2, 17, 70, 128, 2, 2, 32), 1, MEC_PATH_SOLUTION_B),   # shift = 2 atoms, window 4 atoms
    ((2, 40, 60, 64, 7, 7, 64), 2, MEC_PATH_SOLUTION_B),    # cv4-like: 49-atom window, weights streamed
    ((3, 30, 150, 64, 3, 3, 64), 1, "stream"),              # resident-size weights forced to stream
    ((1, 20, 40, 64, 7, 7, 64), 1, MEC_PATH_SOLUTION_B),    # 7 open rows, streamed weights: the 3-D weight
                                                            # box's slabs reach 6 window shifts past K_t
]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", range(len(PS_CASES)))
def test_pair_sweep_kernel(cuda_ok, case, dtype):
    """Atom-major sweep on CTA pairs: every L column read once per
    work item, each atom's MMAs into every open row's accumulator."""
    shape, s, path = PS_CASES[case]
    I, K = make_inputs(shape, dtype, seed=8000 + case)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    stream = path == "stream"
    if stream:
        path = MEC_PATH_SOLUTION_B
        os.environ["MEC_PS_BSTREAM"] = "1"
    try:
        O, g = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=4, return_gemm=True)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("MEC_PS_BSTREAM", None)
    assert g == 4
    check_O(O, ref, dtype, shape[3] * shape[4] * shape[5])
    # same K steps per row as the one-window kernel
    O1 = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=1)
    torch.cuda.synchronize()
    assert torch.equal(O, O1)
    if path == MEC_PATH_SOLUTION_A:  # the paper-literal format fix stores h-n-w-c first
        OL = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=4, sola_fix=MEC_SOLA_FIX_LITERAL)
        torch.cuda.synchronize()
        assert torch.equal(O, OL)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("case", [0, 2, 3, 6, 7])
def test_pair_sweep_balanced_split(cuda_ok, monkeypatch, case, dtype):
    """The pair sweep's balanced split (every pair the same number of (pair tile,
    h) rows, cut at pair-tile boundaries), forced on these small
    shapes (1-2 rows per pair, empty pieces): the same K steps per row as the
    one-window kernel, so bit for bit."""
    shape, s, path = PS_CASES[case]
    I, K = make_inputs(shape, dtype, seed=8100 + case)
    Id, Kd = to_dev(I, dtype), to_dev(K, dtype)
    if path == "stream":
        path = MEC_PATH_SOLUTION_B
        monkeypatch.setenv("MEC_PS_BSTREAM", "1")
    monkeypatch.setenv("MEC_PS_BALANCED", "1")
    O, g = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=4, return_gemm=True)
    torch.cuda.synchronize()
    assert g == 4
    O1 = mec.conv_forward(Id, Kd, s, s, path=path, gemm_kernel=1)
    torch.cuda.synchronize()
    assert torch.equal(O, O1)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    check_O(O, ref, dtype, shape[3] * shape[4] * shape[5])


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_C2_pair_sweep_full_batch_sampled(cuda_ok, dtype):
    """C2 at b64 through the pair sweep (tf32: the automatic choice)."""
    c = "C2" if dtype == "bf16" else "C2_tf32"
    cfg = synth.config(c)
    shape = (cfg["i_n"], cfg["i_h"], cfg["i_w"], cfg["i_c"], cfg["k_h"], cfg["k_w"], cfg["k_c"])
    seed = synth.SEED_BASE + cfg["index"]
    kind = synth.KIND_GRID8 if dtype == "bf16" else synth.KIND_GRID11
    Id = torch.empty(shape[:4], dtype=TDT[dtype], device="cuda")
    Kd = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=TDT[dtype], device="cuda")
    mec.synth_fill(Id, seed, synth.TENSOR_I, kind)
    mec.synth_fill(Kd, seed, synth.TENSOR_K, kind)
    O, g = mec.conv_forward(Id, Kd, 1, 1, gemm_kernel=4, return_gemm=True)
    torch.cuda.synchronize()
    assert g == 4
    K = synth.kernel_tensor(cfg, kind, seed)
    for n in (0, 37, 63):
        I = synth.input_images(cfg, n, 1, kind, seed)
        check_O(O[n:n + 1], oracle.direct_conv(I, K, 1, 1, n_threads=8), dtype, 576)


@pytest.mark.parametrize("name,batch", [("cv12", 3), ("cv5", 2), ("cv1", 2)])
def test_wide_pair_kernel_weights_from_K(cuda_ok, name, batch):
    """Opt-in variant (MEC_WIDE_KMN=1): the CTA-pair kernel reads the weights
    straight from K as an MN-major B operand (no prepared Kt; negative rows of
    a delta-shifted window are TMA zero fill) -- within tolerance of the oracle."""
    i_h, i_w, i_c, k_h, k_w, k_c, s = synth.TABLE2[name]
    shape = (batch, i_h, i_w, i_c, k_h, k_w, k_c)
    I, K = make_inputs(shape, "bf16", seed=6300 + batch)
    ref = oracle.direct_conv(I, K, s, s, n_threads=8)
    os.environ["MEC_WIDE_KMN"] = "1"
    try:
        O, g = mec.conv_forward(to_dev(I, "bf16"), to_dev(K, "bf16"), s, s, path=MEC_PATH_SOLUTION_A,
                                gemm_kernel=3, return_gemm=True)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("MEC_WIDE_KMN", None)
    assert g == 3
    check_O(O, ref, "bf16", k_h * k_w * i_c)
