"""Workload shapes (no method arithmetic).

TABLE2: the paper's 12 benchmark layers, Table 2, as
i_h x i_w x i_c and k_h x k_w x k_c, stride s_h = s_w.
CONFIGS: BASELINE.json "configs" C0..C4 (C4 is a sweep over TABLE2 + three 1x1
layers that Table 2 lacks).
"""
from __future__ import annotations

# name: (i_h, i_w, i_c, k_h, k_w, k_c, s)   -- P:243-254
TABLE2 = {
    "cv1": (227, 227, 3, 11, 11, 96, 4),
    "cv2": (231, 231, 3, 11, 11, 96, 4),
    "cv3": (227, 227, 3, 7, 7, 64, 2),
    "cv4": (224, 224, 64, 7, 7, 64, 2),
    "cv5": (24, 24, 96, 5, 5, 256, 1),
    "cv6": (12, 12, 256, 3, 3, 512, 1),
    "cv7": (224, 224, 3, 3, 3, 64, 1),
    "cv8": (112, 112, 64, 3, 3, 128, 1),
    "cv9": (56, 56, 64, 3, 3, 64, 1),
    "cv10": (28, 28, 128, 3, 3, 128, 1),
    "cv11": (14, 14, 256, 3, 3, 256, 1),
    "cv12": (7, 7, 512, 3, 3, 512, 1),
}

# 1x1 layers for the C4 sweep (BASELINE.json names "1x1" shapes; Table 2 has none).
ONE_BY_ONE = {
    "r50_1x1_256to64": (56, 56, 256, 1, 1, 64, 1),
    "r50_1x1_64to256": (56, 56, 64, 1, 1, 256, 1),
    "g_3a_1x1_192to64": (28, 28, 192, 1, 1, 64, 1),
}


def _mk(name, i_n, t, dtype, **extra):
    i_h, i_w, i_c, k_h, k_w, k_c, s = t
    d = dict(name=name, i_n=i_n, i_h=i_h, i_w=i_w, i_c=i_c, k_h=k_h, k_w=k_w, k_c=k_c,
             s_h=s, s_w=s, dtype=dtype)
    d.update(extra)
    return d


CONFIGS = {
    # C0: paper worked example, Fig. 1 / Fig. 2: 7x7 input, 3x3 kernel, stride 1.
    "C0": _mk("C0_worked_example", 1, (7, 7, 1, 3, 3, 1, 1), "fp32", index=0),
    # C1: AlexNet conv1 (= cv1), batch 32, bf16.
    "C1": _mk("C1_alexnet_conv1", 32, TABLE2["cv1"], "bf16", index=1),
    # C2: VGG-16 conv1_2, batch 64, bf16 and tf32.
    "C2": _mk("C2_vgg16_conv1_2", 64, (224, 224, 64, 3, 3, 64, 1), "bf16", index=2),
    "C2_tf32": _mk("C2_vgg16_conv1_2_tf32", 64, (224, 224, 64, 3, 3, 64, 1), "tf32", index=2),
    # C3: ResNet-50 stage-2 3x3 (= cv9), batch 256, sharded over GPUs.
    "C3": _mk("C3_resnet50_stage2_3x3", 256, TABLE2["cv9"], "bf16", index=3),
}
for _n, _t in list(TABLE2.items()) + list(ONE_BY_ONE.items()):
    CONFIGS[f"C4_{_n}"] = _mk(f"C4_{_n}_b1024", 1024, _t, "bf16", index=4, layer=_n)


def config(name: str, i_n: int | None = None) -> dict:
    """A copy of CONFIGS[name]; i_n overrides the batch.  The C4 sweep's names
    carry the batch actually used (C4_cv4_b128 when i_n = 128)."""
    c = dict(CONFIGS[name])
    if i_n is not None:
        c["i_n"] = i_n
    if "layer" in c:
        c["name"] = f"C4_{c['layer']}_b{c['i_n']}"
    return c
