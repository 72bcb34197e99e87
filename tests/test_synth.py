"""Host side of the counter-based input generator (synth/)."""
import numpy as np

import synth


def test_splitmix64_reference_values():
    # splitmix64 reference sequence for state 0 (Steele, Lea & Flood 2014 / Vigna's C code):
    # outputs 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f
    g = 0x9E3779B97F4A7C15
    x = np.array([0, g, (2 * g) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    got = [int(v) for v in synth.splitmix64(x)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_kinds_ranges_and_exactness():
    v8 = synth.draw(100000, 1, 0, synth.KIND_GRID8)
    assert v8.min() >= -1.0 and v8.max() <= 127 / 128
    assert np.all(v8 * 128 == np.round(v8 * 128))
    # exactly representable in bf16: low 16 bits of the fp32 pattern are zero
    assert np.all((v8.view(np.uint32) & 0xFFFF) == 0)
    v11 = synth.draw(100000, 1, 0, synth.KIND_GRID11)
    assert v11.min() >= -1.0 and v11.max() <= 1023 / 1024
    # exactly representable in tf32: low 13 mantissa bits zero
    assert np.all((v11.view(np.uint32) & 0x1FFF) == 0)
    v24 = synth.draw(100000, 1, 0, synth.KIND_FULL24)
    assert v24.min() >= -1.0 and v24.max() < 1.0
    for v in (v8, v11, v24):
        assert abs(float(v.mean())) < 0.02 and 0.3 < float(v.std()) < 0.7


def test_shards_are_slices_of_global_tensor():
    cfg = synth.config("C1", i_n=8)
    full = synth.input_images(cfg, 0, 8, synth.KIND_GRID8, 5)
    part = synth.input_images(cfg, 3, 2, synth.KIND_GRID8, 5)
    np.testing.assert_array_equal(full[3:5], part)


def test_tensor_ids_and_seeds_differ():
    a = synth.draw(1000, 7, 0, synth.KIND_GRID11)
    b = synth.draw(1000, 7, 1, synth.KIND_GRID11)
    c = synth.draw(1000, 8, 0, synth.KIND_GRID11)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
