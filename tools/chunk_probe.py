"""Probe: C2 (VGG conv1_2 b64) as one mec_conv_forward_ex call versus k calls
on consecutive image chunks sharing one workspace (the chunk's L stays in L2
between its lowering and its GEMMs).  Device time of the whole batch with CUDA
events, L2 flushed before each timed batch.  usage: python tools/chunk_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1706_06873_b200 import mec  # noqa: E402


def main():
    cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
    n, s = cfg["i_n"], cfg["s_h"]
    I = torch.empty((n, cfg["i_h"], cfg["i_w"], cfg["i_c"]), dtype=torch.bfloat16, device="cuda")
    K = torch.empty((cfg["k_h"], cfg["k_w"], cfg["i_c"], cfg["k_c"]), dtype=torch.bfloat16, device="cuda")
    mec.synth_fill(I, 1, 0, 0)
    mec.synth_fill(K, 1, 1, 0)
    o_h, o_w = mec.out_dims(cfg["i_h"], cfg["i_w"], cfg["k_h"], cfg["k_w"], s, s)
    O = torch.empty((n, o_h, o_w, cfg["k_c"]), dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for chunks in (1, 2, 4, 8, 16):
        if n % chunks:
            continue
        c = n // chunks
        shape = (c, cfg["i_h"], cfg["i_w"], cfg["i_c"], cfg["k_h"], cfg["k_w"], cfg["k_c"])
        ws = torch.empty(mec.workspace_bytes(shape, s, s, torch.bfloat16), dtype=torch.uint8, device="cuda")

        def run():
            for j in range(chunks):
                mec.conv_forward(I[j * c:(j + 1) * c], K, s, s, out=O[j * c:(j + 1) * c], workspace=ws)
        for _ in range(3):
            run()
        ts = []
        for _ in range(10):
            mec.l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        out[chunks] = {"ms_median": ts[len(ts) // 2], "ms_min": ts[0], "ws_MB": ws.numel() / 1e6}
        print(chunks, out[chunks], flush=True)
    print(json.dumps({"config": cfg["name"], "chunks": out}))


if __name__ == "__main__":
    main()
