"""Small MEC calls for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): one case per kernel and variant, checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases: C0 (worked example, tf32, Solution A), C1 (AlexNet conv1 b2: lowering
word-table path + h-sweep, 1 issuer), tf32 (a tf32 h-sweep), sweep2 (C3-like
b2: two issuers), window (forced one-window kernel), fused (TMA-box fused),
gather (fused gather, AlexNet conv1 b1), wide (CTA-pair split-K, cv12 b2,
split 2), pair (CTA-pair atom-major sweep, VGG-like), literal (Solution A
literal format fix), pad (virtual padding)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1706_06873_b200 import mec  # noqa: E402
from paper_1706_06873_b200._lib import (MEC_PATH_FUSED, MEC_PATH_SOLUTION_A, MEC_PATH_SOLUTION_B,  # noqa: E402
                                        MEC_SOLA_FIX_LITERAL)

T = {"bf16": torch.bfloat16, "tf32": torch.float32}


def run(name, shape, s, dtype, tol_rel, **kw):
    i_n, i_h, i_w, i_c, k_h, k_w, k_c = shape
    cfg = dict(i_h=i_h, i_w=i_w, i_c=i_c, k_h=k_h, k_w=k_w, k_c=k_c)
    kind = synth.KIND_GRID8 if dtype == "bf16" else synth.KIND_GRID11
    I = synth.input_images(cfg, 0, i_n, kind, 11)
    K = synth.kernel_tensor(cfg, kind, 11)
    pad = kw.get("pad_h", 0)
    ref = oracle.direct_conv(np.pad(I, ((0, 0), (pad, pad), (pad, pad), (0, 0))) if pad else I, K, s, s, n_threads=8)
    O = mec.conv_forward(torch.from_numpy(I).cuda().to(T[dtype]), torch.from_numpy(K).cuda().to(T[dtype]), s, s, **kw)
    torch.cuda.synchronize()
    err = float(np.abs(O.float().cpu().numpy() - ref).max()) / max(float(np.abs(ref).max()), 1e-30)
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err <= tol_rel, name


CASES = {
    "C0": lambda: run("C0", (1, 7, 7, 1, 3, 3, 1), 1, "tf32", 1e-3, path=MEC_PATH_SOLUTION_A),
    "C1": lambda: run("C1", (2, 227, 227, 3, 11, 11, 96), 4, "bf16", 2e-2),
    "tf32": lambda: run("tf32", (2, 40, 40, 16, 3, 3, 32), 1, "tf32", 1e-2),
    "sweep2": lambda: run("sweep2", (2, 56, 56, 64, 3, 3, 64), 1, "bf16", 2e-2),
    "window": lambda: run("window", (2, 30, 31, 16, 3, 3, 40), 1, "bf16", 2e-2, gemm_kernel=1),
    "fused": lambda: run("fused", (2, 30, 40, 64, 3, 3, 64), 1, "bf16", 2e-2, path=MEC_PATH_FUSED),
    "gather": lambda: run("gather", (1, 227, 227, 3, 11, 11, 96), 4, "bf16", 2e-2, path=MEC_PATH_FUSED),
    "wide": lambda: run("wide", (2, 7, 7, 512, 3, 3, 512), 1, "bf16", 2e-2, path=MEC_PATH_SOLUTION_A,
                        gemm_kernel=3, split_k=2),
    "pair": lambda: run("pair", (2, 20, 150, 64, 3, 3, 64), 1, "tf32", 1e-2, path=MEC_PATH_SOLUTION_B,
                        gemm_kernel=4),
    "literal": lambda: run("literal", (3, 23, 21, 6, 3, 3, 24), 2, "bf16", 2e-2, path=MEC_PATH_SOLUTION_A,
                           sola_fix=MEC_SOLA_FIX_LITERAL),
    "pad": lambda: run("pad", (2, 14, 14, 64, 3, 3, 64), 1, "bf16", 2e-2, pad_h=1, pad_w=1),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
    print("sanitize cases ok:", " ".join(names))
