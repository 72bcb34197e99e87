"""PCIe copy probe: pinned H2D and D2H bandwidth alone and concurrently (the e2e bound)."""
import json
import sys

import torch


def timed(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main(h2d_bytes=9963264, d2h_bytes=18585600):
    hi = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
    ho = torch.empty(d2h_bytes, dtype=torch.uint8).pin_memory()
    di = torch.empty(h2d_bytes, dtype=torch.uint8, device="cuda")
    do = torch.empty(d2h_bytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2d = timed(lambda: di.copy_(hi, non_blocking=True))
    d2h = timed(lambda: ho.copy_(do, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    bo = timed(both)

    def chunked(n):
        hb, ob = h2d_bytes // n // 16 * 16, d2h_bytes // n // 16 * 16

        def f():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            for c in range(n):
                with torch.cuda.stream(s1):
                    di[c * hb:(c + 1) * hb].copy_(hi[c * hb:(c + 1) * hb], non_blocking=True)
                with torch.cuda.stream(s2):
                    ho[c * ob:(c + 1) * ob].copy_(do[c * ob:(c + 1) * ob], non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        torch.cuda.synchronize()
        torch.cuda._sleep(4_000_000)
        return timed(f, reps=5)

    chunk_ms = {n: chunked(n) for n in (1, 4, 8)}
    print(json.dumps({"h2d_ms": h2d, "h2d_GBps": h2d_bytes / h2d / 1e6, "d2h_ms": d2h,
                      "d2h_GBps": d2h_bytes / d2h / 1e6, "both_concurrent_ms": bo,
                      "serial_ms": h2d + d2h, "both_chunked_ms": chunk_ms}))




def host_enqueue_probe():
    """Host-side time of one enqueue of the e2e call per chunk count (GPU left to drain)."""
    import time

    from paper_1706_06873_b200 import mec
    I_h = torch.zeros((32, 227, 227, 3), dtype=torch.bfloat16).pin_memory()
    K_h = torch.zeros((11, 11, 3, 96), dtype=torch.bfloat16).pin_memory()
    O_h = torch.empty((32, 55, 55, 96), dtype=torch.bfloat16).pin_memory()
    Id, Kd = I_h.cuda(), K_h.cuda()
    Od = torch.empty((32, 55, 55, 96), dtype=torch.bfloat16, device="cuda")
    out = {}
    for nch in (1, 2, 4, 8):
        sc = torch.empty(mec.host_scratch_bytes(32, 227, 227, 3, 11, 11, 96, 4, 4, torch.bfloat16, nch),
                         dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mec.conv_forward_host(I_h, K_h, 4, 4, out=O_h, n_chunks=nch, scratch=sc)
            ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        out[f"host_call_us_chunks{nch}"] = sorted(ts)[5] * 1e6
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mec.conv_forward(Id, Kd, 4, 4, out=Od)
        ts.append(time.perf_counter() - t0)
    out["device_call_us"] = sorted(ts)[5] * 1e6
    print(json.dumps(out))



def library_presleep():
    """mec_conv_forward_host timed with the GPU held back until the host has enqueued everything."""
    from paper_1706_06873_b200 import mec
    I_h = torch.zeros((32, 227, 227, 3), dtype=torch.bfloat16).pin_memory()
    K_h = torch.zeros((11, 11, 3, 96), dtype=torch.bfloat16).pin_memory()
    O_h = torch.empty((32, 55, 55, 96), dtype=torch.bfloat16).pin_memory()
    out = {}
    for nch in (1, 2, 4, 8, 16, 32):
        sc = torch.empty(mec.host_scratch_bytes(32, 227, 227, 3, 11, 11, 96, 4, 4, torch.bfloat16, nch),
                         dtype=torch.uint8, device="cuda")
        r = {}
        for sleep in (0, 1):
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                if sleep:
                    torch.cuda._sleep(4_000_000)
                a.record()
                mec.conv_forward_host(I_h, K_h, 4, 4, out=O_h, n_chunks=nch, scratch=sc)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            r["presleep" if sleep else "plain"] = sorted(ts)[3]
        out[nch] = r
    print(json.dumps(out))


def pipeline_emulation(nch=8):
    """The e2e pipeline rebuilt from torch streams around the device call, with timing events
    at every stage (to see where the host-buffer call loses time)."""
    from paper_1706_06873_b200 import mec
    N = 32
    I_h = torch.zeros((N, 227, 227, 3), dtype=torch.bfloat16).pin_memory()
    K_h = torch.zeros((11, 11, 3, 96), dtype=torch.bfloat16).pin_memory()
    O_h = torch.empty((N, 55, 55, 96), dtype=torch.bfloat16).pin_memory()
    Id = torch.empty_like(I_h, device="cuda")
    Kd = torch.empty_like(K_h, device="cuda")
    Od = torch.empty_like(O_h, device="cuda")
    sh, sc, so = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    b = N // nch
    Ids = [torch.empty((b, 227, 227, 3), dtype=torch.bfloat16, device="cuda") for _ in range(nch)]
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    res = {}
    for it in range(3):
        ev = {k: [E() for _ in range(nch)] for k in ("in", "comp", "out")}
        t0 = E()
        cur = torch.cuda.current_stream()
        torch.cuda.synchronize()
        torch.cuda._sleep(4_000_000)  # ~2 ms: the whole enqueue lands before the GPU starts
        t0.record(cur)
        for s in (sh, sc, so):
            s.wait_stream(cur)
        with torch.cuda.stream(sh):
            Kd.copy_(K_h, non_blocking=True)
        for c in range(nch):
            sl = slice(c * b, (c + 1) * b)
            with torch.cuda.stream(sh):
                Ids[c].copy_(I_h[sl], non_blocking=True)
                ev["in"][c].record(sh)
            sc.wait_event(ev["in"][c])
            with torch.cuda.stream(sc):
                mec.conv_forward(Ids[c], Kd, 4, 4, out=Od[sl])
                ev["comp"][c].record(sc)
            so.wait_event(ev["comp"][c])
            with torch.cuda.stream(so):
                O_h[sl].copy_(Od[sl], non_blocking=True)
                ev["out"][c].record(so)
        cur.wait_stream(so)
        t1 = E()
        t1.record(cur)
        torch.cuda.synchronize()
        res = {"total_ms": t0.elapsed_time(t1)}
        for k in ev:
            res[k] = [round(t0.elapsed_time(e), 3) for e in ev[k]]
    print(json.dumps(res))


if __name__ == "__main__":
    if "--enqueue" in sys.argv:
        host_enqueue_probe()
    elif "--presleep" in sys.argv:
        library_presleep()
    elif "--emulate" in sys.argv:
        pipeline_emulation(int(sys.argv[2]) if len(sys.argv) > 2 else 8)
    else:
        main(*[int(a) for a in sys.argv[1:]])
