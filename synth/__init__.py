"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the MEC method: only a counter-based
random generator and the workload shapes of BASELINE.json / PAPER.md Table 2.
Both sides draw the same numbers: the host evaluates the generator here with
numpy; the device evaluates the same formula in its own CUDA kernel
(``mec_synth_fill`` in paper_1706_06873_b200/csrc/synth.cu, written separately).
A test (tests/test_gpu_parity.py::test_device_generator_matches_host) checks
the two agree bit for bit.

Generator ("input recipe"):
  x   = seed XOR (tensor_id << 56) XOR global_linear_index      (uint64)
  z   = splitmix64(x)
  kinds:
    GRID8  (bf16 / fp32):  v = int8(z >> 56) / 128          in [-1, 127/128]
    GRID11 (fp32 / tf32):  v = ((z >> 53) - 1024) / 1024    in [-1, 1023/1024]
    FULL24 (fp32):         v = ((z >> 40) - 2^23) / 2^23    in [-1, 1)
GRID8 values are exact in bf16, GRID11 values exact in tf32, so on the grid
kinds the GPU's only error is its accumulation order (and the bf16 rounding
of O).  global_linear_index uses the GLOBAL image index n, so a rank's shard
is a slice of the single-GPU tensor.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 170606873  # arXiv id 1706.06873; seed = SEED_BASE + config index
TENSOR_I = 0
TENSOR_K = 1

KIND_GRID8 = 0
KIND_GRID11 = 1
KIND_FULL24 = 2

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of (x + golden gamma), vectorised over uint64."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def draw(count: int, seed: int, tensor_id: int, kind: int, index_offset: int = 0) -> np.ndarray:
    """Return `count` float32 values for global indices [index_offset, index_offset+count)."""
    idx = np.arange(index_offset, index_offset + count, dtype=np.uint64)
    x = np.uint64(seed) ^ (np.uint64(tensor_id) << np.uint64(56)) ^ idx
    z = splitmix64(x)
    if kind == KIND_GRID8:
        v = (z >> np.uint64(56)).astype(np.uint8).view(np.int8).astype(np.float32) / np.float32(128.0)
    elif kind == KIND_GRID11:
        v = ((z >> np.uint64(53)).astype(np.int64) - 1024).astype(np.float32) / np.float32(1024.0)
    elif kind == KIND_FULL24:
        v = ((z >> np.uint64(40)).astype(np.int64) - (1 << 23)).astype(np.float32) / np.float32(1 << 23)
    else:
        raise ValueError(f"unknown kind {kind}")
    return v.astype(np.float32)


def tensor(shape, seed: int, tensor_id: int, kind: int, index_offset: int = 0) -> np.ndarray:
    """A float32 array of `shape` filled by `draw` (row-major global indices)."""
    n = int(np.prod(shape))
    return draw(n, seed, tensor_id, kind, index_offset).reshape(shape)


def input_images(cfg: dict, n_begin: int, n_count: int, kind: int, seed: int) -> np.ndarray:
    """Images [n_begin, n_begin+n_count) of the config's I (NHWC), float32."""
    per = cfg["i_h"] * cfg["i_w"] * cfg["i_c"]
    return tensor((n_count, cfg["i_h"], cfg["i_w"], cfg["i_c"]), seed, TENSOR_I, kind,
                  index_offset=n_begin * per)


def kernel_tensor(cfg: dict, kind: int, seed: int) -> np.ndarray:
    """The config's K (k_h, k_w, i_c, k_c), float32."""
    return tensor((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), seed, TENSOR_K, kind)


from .configs import CONFIGS, ONE_BY_ONE, TABLE2, config  # noqa: E402,F401
