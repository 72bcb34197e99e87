"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every test here is CPU-only.  Each pin is something other than the oracle
itself: numbers printed in PAPER.md (tests/golden/*), closed forms, library
routines (torch.nn.functional.conv2d in fp64, numpy matmul / sliding windows),
invariants and special cases.  A dropped term, wrong sign, wrong index or
transposed operand in the oracle fails at least one of them.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from mec_testutil import golden, read_kv

WE = read_kv("worked_example.txt")


def ramp_image():
    """I[h, w] = 7h + w on the 7x7 worked example (values are ours; Fig.1's are lost)."""
    return np.array([[7 * h + w for w in range(7)] for h in range(7)], dtype=np.float64)


def torch_conv(I, K, s_h, s_w):
    """Library reference: cross-correlation via torch conv2d in float64, NHWC in/out."""
    x = torch.from_numpy(np.ascontiguousarray(I)).permute(0, 3, 1, 2)
    k = torch.from_numpy(np.ascontiguousarray(K)).permute(3, 2, 0, 1)
    return F.conv2d(x, k, stride=(s_h, s_w)).permute(0, 2, 3, 1).contiguous().numpy()


# --------------------------------------------------------------- Eq. (1)

def test_eq1_worked_example_dims():
    # Fig. 1 caption: 7x7 input, 3x3 kernel, stride 1 -> 5x5
    assert oracle.out_dims((1, WE["i_h"], WE["i_w"], 1, WE["k_h"], WE["k_w"], 1), WE["s"], WE["s"]) == (
        WE["o"], WE["o"])


def test_eq1_floor_pinned_by_table3_cv4():
    # Table 3 cv4: 224x224x64, 7x7x64, s=2.  Only o = floor(217/2)+1 = 109
    # reproduces the printed 142.1 / 41.7 MiB (ceil would give 144.8 / 42.1).
    shp = (1, 224, 224, 64, 7, 7, 64)
    assert oracle.out_dims(shp, 2, 2) == (109, 109)
    mib = 4 / 2**20
    assert abs(oracle.elems_L_im2col(shp, 2, 2) * mib - 142.1) < 0.05
    assert abs(oracle.elems_L_mec(shp, 2, 2) * mib - 41.7) < 0.05


@pytest.mark.parametrize("bad", [
    ((1, 2, 7, 1, 3, 3, 1), 1, 1),   # i_h < k_h
    ((1, 7, 2, 1, 3, 3, 1), 1, 1),   # i_w < k_w
    ((1, 7, 7, 1, 3, 3, 1), 0, 1),   # s_h < 1
    ((0, 7, 7, 1, 3, 3, 1), 1, 1),   # empty batch
    ((1, 7, 7, 1, 3, 3, 0), 1, 1),   # no output channels
])
def test_eq1_rejects_invalid(bad):
    with pytest.raises(ValueError):
        oracle.out_dims(*bad)


# ----------------------------------------------- worked example (Fig. 1, 2)

def test_worked_example_sizes():
    shp = (1, 7, 7, 1, 3, 3, 1)
    C = oracle.im2col(ramp_image().reshape(1, 7, 7, 1), 3, 3, 1, 1)
    assert C.shape == (WE["im2col_rows"], WE["im2col_cols"])
    L = oracle.lower(ramp_image().reshape(1, 7, 7, 1), 3, 3, 1, 1)
    assert L.reshape(5, -1).shape == (WE["mec_rows"], WE["mec_cols"])
    n_mec, n_im2col = oracle.elems_L_mec(shp, 1, 1), oracle.elems_L_im2col(shp, 1, 1)
    assert (n_mec, n_im2col) == (105, 225)
    # "54% smaller": exactly 1 - 105/225 = 53.3% (reading Q12)
    assert abs(100 * (1 - n_mec / n_im2col) - WE["mec_smaller_pct"]) < 1.0


def test_worked_example_horizontal_partitions():
    # row 0 of L is A = I[0:7,0:3], row 1 is B = I[0:7,1:4] (each 7x3, row-major)
    I2 = ramp_image()
    L = oracle.lower(I2.reshape(1, 7, 7, 1), 3, 3, 1, 1).reshape(5, 21)
    a0, a1 = WE["partition_A_cols"]
    b0, b1 = WE["partition_B_cols"]
    np.testing.assert_array_equal(L[0], I2[0:7, a0:a1].reshape(-1))
    np.testing.assert_array_equal(L[1], I2[0:7, b0:b1].reshape(-1))
    for w in range(5):  # and so on for C, D, E
        np.testing.assert_array_equal(L[w], I2[0:7, w:w + 3].reshape(-1))


def test_worked_example_vertical_partitions_give_output_rows():
    # P = L[0:5,0:9], Q = L[0:5,3:12], ..., shift s_h k_w = 3, ld = 21;
    # output row h = partition_h x K (K as k_h k_w x 1).  numpy matmul, not the oracle's GEMM.
    rng = np.random.default_rng(0)
    I2 = rng.standard_normal((7, 7))
    K2 = rng.standard_normal((3, 3))
    L = oracle.lower(I2.reshape(1, 7, 7, 1), 3, 3, 1, 1).reshape(5, WE["ld"])
    O_ref = torch_conv(I2.reshape(1, 7, 7, 1), K2.reshape(3, 3, 1, 1), 1, 1).reshape(5, 5)
    p0, p1 = WE["partition_P_cols"]
    q0, q1 = WE["partition_Q_cols"]
    np.testing.assert_allclose(L[:, p0:p1] @ K2.reshape(9), O_ref[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(L[:, q0:q1] @ K2.reshape(9), O_ref[1], rtol=1e-12, atol=1e-12)
    for h in range(WE["n_gemm"]):
        sh = WE["vertical_shift"] * h
        np.testing.assert_allclose(L[:, sh:sh + 9] @ K2.reshape(9), O_ref[h], rtol=1e-12, atol=1e-12)


def test_ramp_closed_form_all_paths():
    # I[h,w] = 7h + w, K = ones(3x3): O[h,w] = sum_{a,b} 7(h+a) + (w+b) = 9(7h+w) + 72
    I = ramp_image().reshape(1, 7, 7, 1)
    K = np.ones((3, 3, 1, 1))
    expect = np.array([[9 * (7 * h + w) + 72 for w in range(5)] for h in range(5)], dtype=np.float64)
    assert expect[0, 0] == 72 and expect[4, 4] == 360
    np.testing.assert_array_equal(oracle.direct_conv(I, K, 1, 1)[0, :, :, 0], expect)
    np.testing.assert_array_equal(oracle.vanilla_mec(ramp_image(), np.ones((3, 3)), 1, 1), expect)
    np.testing.assert_array_equal(oracle.conv_solA(I, K, 1, 1)[0, :, :, 0], expect)
    np.testing.assert_array_equal(oracle.conv_solB(I, K, 1, 1)[0, :, :, 0], expect)
    O, path = oracle.mec(I, K, 1, 1)
    assert path == 1  # o_w = 5 <= 100 and #O = 25 <= #L = 105
    np.testing.assert_array_equal(O[0, :, :, 0], expect)


@pytest.mark.parametrize("seed", range(6))
def test_linear_image_closed_form(seed):
    # I = alpha h + beta w + gamma c + delta n, K = 1: with S(k) = k(k-1)/2,
    # O[n,h,w,:] = k_h k_w i_c (alpha h s_h + beta w s_w + delta n)
    #            + alpha k_w i_c S(k_h) + beta k_h i_c S(k_w) + gamma k_h k_w S(i_c)
    rng = np.random.default_rng(100 + seed)
    i_n, i_c, k_c = rng.integers(1, 4, 3)
    k_h, k_w = rng.integers(1, 6, 2)
    s_h, s_w = rng.integers(1, 5, 2)
    i_h, i_w = k_h + rng.integers(0, 9), k_w + rng.integers(0, 9)
    al, be, ga, de = 7.0, -3.0, 0.5, 100.0
    n, h, w, c = np.meshgrid(np.arange(i_n), np.arange(i_h), np.arange(i_w), np.arange(i_c), indexing="ij")
    I = al * h + be * w + ga * c + de * n
    K = np.ones((k_h, k_w, i_c, k_c))
    O = oracle.direct_conv(I, K, int(s_h), int(s_w))
    o_h, o_w = (i_h - k_h) // s_h + 1, (i_w - k_w) // s_w + 1
    S = lambda k: k * (k - 1) / 2  # noqa: E731
    nn, hh, ww = np.meshgrid(np.arange(i_n), np.arange(o_h), np.arange(o_w), indexing="ij")
    expect = (k_h * k_w * i_c * (al * hh * s_h + be * ww * s_w + de * nn)
              + al * k_w * i_c * S(k_h) + be * k_h * i_c * S(k_w) + ga * k_h * k_w * S(i_c))
    np.testing.assert_allclose(O, np.repeat(expect[..., None], k_c, axis=3), rtol=1e-12, atol=1e-9)


# -------------------------------------------------- library cross-checks

def random_cases(n_cases, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n_cases):
        i_n, i_c, k_c = (int(v) for v in rng.integers(1, 4, 3))
        k_h, k_w = (int(v) for v in rng.integers(1, 6, 2))
        s_h, s_w = (int(v) for v in rng.integers(1, 5, 2))
        i_h, i_w = k_h + int(rng.integers(0, 10)), k_w + int(rng.integers(0, 10))
        I = rng.standard_normal((i_n, i_h, i_w, i_c))
        K = rng.standard_normal((k_h, k_w, i_c, k_c))
        yield I, K, s_h, s_w


@pytest.mark.parametrize("chunk", range(4))
def test_all_oracle_convs_match_torch_conv2d(chunk):
    # 4 x 60 random tiny shapes incl. non-divisible strides and s > k
    for I, K, s_h, s_w in random_cases(60, 1000 + chunk):
        ref = torch_conv(I, K, s_h, s_w)
        D = oracle.direct_conv(I, K, s_h, s_w)
        np.testing.assert_allclose(D, ref, rtol=1e-12, atol=1e-12)
        B = oracle.conv_solB(I, K, s_h, s_w, n_threads=2)
        # Solution B accumulates j = (a k_w + b) i_c + ci in the same order as direct conv
        np.testing.assert_array_equal(B, D)
        O, path = oracle.mec(I, K, s_h, s_w, T=100)
        np.testing.assert_array_equal(O, D)
        if oracle.elems_O(I.shape + (K.shape[0], K.shape[1], K.shape[3]), s_h, s_w) <= \
                oracle.elems_L_mec(I.shape + (K.shape[0], K.shape[1], K.shape[3]), s_h, s_w):
            np.testing.assert_array_equal(oracle.conv_solA(I, K, s_h, s_w), D)
        # im2col (Fig.1(b)) times K with numpy's matmul
        C = oracle.im2col(I, K.shape[0], K.shape[1], s_h, s_w)
        np.testing.assert_allclose((C @ K.reshape(-1, K.shape[3])).reshape(ref.shape), ref,
                                   rtol=1e-12, atol=1e-12)


def test_threshold_forces_both_solutions_equal():
    # both solutions "perform the same number of floating point multiplications"
    for I, K, s_h, s_w in random_cases(40, 77):
        shp = I.shape + (K.shape[0], K.shape[1], K.shape[3])
        if oracle.elems_O(shp, s_h, s_w) > oracle.elems_L_mec(shp, s_h, s_w):
            continue
        OA, pA = oracle.mec(I, K, s_h, s_w, T=10**9)
        OB, pB = oracle.mec(I, K, s_h, s_w, T=-1)
        assert (pA, pB) == (1, 2)
        np.testing.assert_array_equal(OA, OB)


def test_vanilla_mec_equals_algorithm2_special_case():
    # P:139 / P:201: Algorithm 2 extends Algorithm 1; at i_n = i_c = k_c = 1 they agree.
    rng = np.random.default_rng(5)
    for _ in range(40):
        k_h, k_w = (int(v) for v in rng.integers(1, 6, 2))
        s_h, s_w = (int(v) for v in rng.integers(1, 4, 2))
        i_h, i_w = k_h + int(rng.integers(0, 8)), k_w + int(rng.integers(0, 8))
        I2 = rng.standard_normal((i_h, i_w))
        K2 = rng.standard_normal((k_h, k_w))
        V = oracle.vanilla_mec(I2, K2, s_h, s_w)
        B = oracle.conv_solB(I2.reshape(1, i_h, i_w, 1), K2.reshape(k_h, k_w, 1, 1), s_h, s_w)
        np.testing.assert_array_equal(V, B[0, :, :, 0])
        np.testing.assert_allclose(V, torch_conv(I2[None, :, :, None], K2[:, :, None, None], s_h, s_w)[0, :, :, 0],
                                   rtol=1e-12, atol=1e-12)


def test_one_by_one_is_plain_gemm_and_lowering_is_hw_swap():
    rng = np.random.default_rng(9)
    I = rng.standard_normal((2, 5, 6, 7))
    K = rng.standard_normal((1, 1, 7, 4))
    O = oracle.direct_conv(I, K, 1, 1)
    np.testing.assert_allclose(O.reshape(-1, 4), I.reshape(-1, 7) @ K.reshape(7, 4), rtol=1e-12, atol=1e-12)
    L = oracle.lower(I, 1, 1, 1, 1)  # (n, o_w=w, i_h=h, 1, c)
    np.testing.assert_array_equal(L[:, :, :, 0, :], I.transpose(0, 2, 1, 3))


def test_kernel_equal_to_image_is_dot_products():
    rng = np.random.default_rng(10)
    I = rng.standard_normal((3, 4, 5, 2))
    K = rng.standard_normal((4, 5, 2, 3))
    O = oracle.direct_conv(I, K, 1, 1)
    assert O.shape == (3, 1, 1, 3)
    np.testing.assert_allclose(O[:, 0, 0, :], np.tensordot(I, K, axes=([1, 2, 3], [0, 1, 2])),
                               rtol=1e-12, atol=1e-12)
    L = oracle.lower(I, 4, 5, 1, 1)  # o_w = 1: L[n,0] = I[n] (row-major identical)
    np.testing.assert_array_equal(L.reshape(3, -1), I.reshape(3, -1))


# -------------------------------------------------------------- lowering

@pytest.mark.parametrize("dtype", [np.uint16, np.uint32, np.float64])
def test_lowering_bitexact_vs_numpy_sliding_window(dtype):
    rng = np.random.default_rng(11)
    for _ in range(60):
        i_n, i_c = (int(v) for v in rng.integers(1, 4, 2))
        k_h, k_w = (int(v) for v in rng.integers(1, 6, 2))
        s_h, s_w = (int(v) for v in rng.integers(1, 5, 2))
        i_h, i_w = k_h + int(rng.integers(0, 8)), k_w + int(rng.integers(0, 8))
        if dtype == np.float64:
            I = rng.standard_normal((i_n, i_h, i_w, i_c))
        else:  # arbitrary bit patterns, incl. NaN/Inf encodings
            I = rng.integers(0, np.iinfo(dtype).max, (i_n, i_h, i_w, i_c), dtype=dtype, endpoint=True)
        L = oracle.lower(I, k_h, k_w, s_h, s_w)
        win = np.lib.stride_tricks.sliding_window_view(I, k_w, axis=2)[:, :, ::s_w]  # (n,h,o_w,c,k_w)
        ref = win.transpose(0, 2, 1, 4, 3)  # (n, o_w, h, k_w, c)
        assert L.shape == ref.shape
        np.testing.assert_array_equal(L.view(np.uint8), np.ascontiguousarray(ref).view(np.uint8))


def test_lowering_horizontal_redundancy_invariant():
    # MEC keeps im2col's horizontal redundancy: strips of neighbouring w overlap by k_w - s_w
    rng = np.random.default_rng(12)
    I = rng.standard_normal((2, 9, 17, 3))
    for k_w, s_w in [(5, 1), (5, 2), (7, 3), (3, 4)]:
        L = oracle.lower(I, 3, k_w, 1, s_w)
        for b in range(k_w - s_w):
            np.testing.assert_array_equal(L[:, 1:, :, b, :], L[:, :-1, :, b + s_w, :])


# ------------------------------------------------------- memory analysis

def test_table3_mem_column():
    from synth.configs import TABLE2

    rows = []
    with open(golden("table3_resnet101.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if line:
                rows.append(line)
    mib = 4 / 2**20  # fp32, MB read as MiB
    tot_conv = tot_mec = 0.0
    for name, weight, conv_mb, mec_mb in rows:
        if name == "SUM":
            assert abs(tot_conv - float(conv_mb)) < 0.15
            assert abs(tot_mec - float(mec_mb)) < 0.15
            assert round(tot_conv / tot_mec, 1) == 3.2  # RATIO row
            continue
        i_h, i_w, i_c, k_h, k_w, k_c, s = TABLE2[name]
        shp = (1, i_h, i_w, i_c, k_h, k_w, k_c)  # mini-batch 1 on Mobile
        conv = oracle.elems_L_im2col(shp, s, s) * mib * int(weight)
        mec = oracle.elems_L_mec(shp, s, s) * mib * int(weight)
        # +-0.1 MiB: cv9's printed MEC value 6.7 is 6.645 by the closed form (reading Q16)
        assert abs(conv - float(conv_mb)) < 0.1, name
        assert abs(mec - float(mec_mb)) < 0.1, name
        tot_conv += conv
        tot_mec += mec


@pytest.mark.parametrize("i_h,k_h,s_h", [(7, 3, 1), (227, 11, 4), (25, 5, 2), (56, 3, 1), (12, 3, 3), (9, 1, 2)])
def test_eq4_difference_closed_form(i_h, k_h, s_h):
    # Eq. (4), with i_c for the printed k_c (reading Q2); exact when s_h | (i_h - k_h)
    assert (i_h - k_h) % s_h == 0
    i_n, i_w, i_c, k_w, k_c, s_w = 2, 13, 3, 4, 5, 3
    shp = (i_n, i_h, i_w, i_c, k_h, k_w, k_c)
    _, o_w = oracle.out_dims(shp, s_h, s_w)
    R = oracle.elems_L_im2col(shp, s_h, s_w) - oracle.elems_L_mec(shp, s_h, s_w)
    # R = i_n i_c o_w k_w (i_h - k_h)(k_h / s_h - 1), multiplied through by s_h
    assert R * s_h == i_n * i_c * o_w * k_w * (i_h - k_h) * (k_h - s_h)


def test_eq4_not_always_nonnegative_when_stride_does_not_divide():
    # Reading Q14: "always reduces ... as long as k_h > s_h" needs s_h | (i_h - k_h)
    shp = (1, 4, 4, 1, 3, 3, 1)
    assert oracle.out_dims(shp, 2, 2) == (1, 1)
    assert oracle.elems_L_mec(shp, 2, 2) > oracle.elems_L_im2col(shp, 2, 2)


# ------------------------------------------------------- path selection

# Alg.2 l.8 evaluated by hand (o_w; #O vs #L with i_n cancelled: o_h k_c vs i_h k_w i_c).
PATH_CASES = [
    # name, shape, s, expected path, why
    ("C0", (1, 7, 7, 1, 3, 3, 1), 1, 1, "o_w 5; 5*1 <= 7*3*1"),
    ("C1 cv1", (32, 227, 227, 3, 11, 11, 96), 4, 1, "o_w 55; 55*96=5280 <= 227*11*3=7491"),
    ("C2", (64, 224, 224, 64, 3, 3, 64), 1, 2, "o_w 222 > 100"),
    ("C3 cv9", (256, 56, 56, 64, 3, 3, 64), 1, 1, "o_w 54; 54*64 <= 56*3*64"),
    ("cv3", (1, 227, 227, 3, 7, 7, 64), 2, 2, "o_w 111 > 100"),
    ("cv5", (1, 24, 24, 96, 5, 5, 256), 1, 1, "o_w 20; 20*256=5120 <= 24*5*96=11520"),
    ("cv7", (1, 224, 224, 3, 3, 3, 64), 1, 2, "o_w 222 > 100"),
    ("small #L", (1, 30, 30, 1, 3, 3, 64), 1, 2, "o_w 28 but 28*64=1792 > 30*3*1=90"),
]


@pytest.mark.parametrize("name,shape,s,expect,why", PATH_CASES)
def test_select_path_by_hand(name, shape, s, expect, why):
    assert oracle.select_path(shape, s, s, 100) == expect, why


def test_select_path_threshold_inclusive():
    shp = (1, 102, 102, 4, 3, 3, 4)  # o_w = 100, #O <= #L
    assert oracle.select_path(shp, 1, 1, 100) == 1
    assert oracle.select_path(shp, 1, 1, 99) == 2


def test_solution_A_unavailable_when_O_larger_than_L():
    rng = np.random.default_rng(3)
    I = rng.standard_normal((1, 6, 6, 1))
    K = rng.standard_normal((3, 3, 1, 8))  # #O = 4*4*8 = 128 > #L = 4*6*3 = 72
    with pytest.raises(ValueError):
        oracle.conv_solA(I, K, 1, 1)
    O, path = oracle.mec(I, K, 1, 1, T=100)
    assert path == 2
    np.testing.assert_allclose(O, torch_conv(I, K, 1, 1), rtol=1e-12, atol=1e-12)


def test_multithreaded_equals_single_threaded():
    rng = np.random.default_rng(4)
    I = rng.standard_normal((7, 12, 11, 3))
    K = rng.standard_normal((3, 4, 3, 5))
    for t in (1, 3, 8):
        np.testing.assert_array_equal(oracle.direct_conv(I, K, 2, 1, n_threads=t),
                                      oracle.direct_conv(I, K, 2, 1, n_threads=1))
        np.testing.assert_array_equal(oracle.conv_solB(I, K, 2, 1, n_threads=t),
                                      oracle.conv_solB(I, K, 2, 1, n_threads=1))
