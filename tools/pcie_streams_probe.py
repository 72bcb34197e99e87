"""PCIe probe for the e2e bound of C2 (VGG conv1_2 b64: 411 MB in, 404 MB out):
pinned H2D / D2H bandwidth with the bytes split over 1, 2 or 4 concurrent
streams (several DMA engines), alone and both directions at once."""
import json

import torch


def timed(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main(h2d_bytes=411115520, d2h_bytes=403734528):
    hi = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
    ho = torch.empty(d2h_bytes, dtype=torch.uint8).pin_memory()
    di = torch.empty(h2d_bytes, dtype=torch.uint8, device="cuda")
    do = torch.empty(d2h_bytes, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(8)]
    out = {}

    def split(ns, h2d, d2h, chunks=1):
        def f():
            cur = torch.cuda.current_stream()
            for s in streams[:2 * ns]:
                s.wait_stream(cur)
            for d, (dst, src, n) in enumerate(((di, hi, h2d_bytes), (ho, do, d2h_bytes))):
                if (d == 0 and not h2d) or (d == 1 and not d2h):
                    continue
                parts = ns * chunks
                step = n // parts // 16 * 16
                for k in range(parts):
                    lo, hi_ = k * step, (n if k == parts - 1 else (k + 1) * step)
                    with torch.cuda.stream(streams[d * ns + k % ns]):
                        dst[lo:hi_].copy_(src[lo:hi_], non_blocking=True)
            for s in streams[:2 * ns]:
                cur.wait_stream(s)
        return timed(f)

    for ns in (1, 2, 4):
        t_in = split(ns, True, False)
        t_out = split(ns, False, True)
        t_both = split(ns, True, True)
        t_both16 = split(ns, True, True, chunks=max(1, 16 // ns))
        out[f"streams_{ns}"] = {"h2d_ms": t_in, "h2d_GBps": h2d_bytes / t_in / 1e6, "d2h_ms": t_out,
                                "d2h_GBps": d2h_bytes / t_out / 1e6, "both_ms": t_both,
                                "both_16chunks_ms": t_both16}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
