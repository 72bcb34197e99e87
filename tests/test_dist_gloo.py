"""Multi-process (gloo, world_size 2, CPU) tests of the batch-sharded driver
(paper_1706_06873_b200/dist.py): image sharding, the single broadcast of K,
max-over-ranks timing, and that per-rank shards of the synthetic input are
slices of the single-process tensor (so sharded O == single-GPU O)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(ws), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import oracle
        import synth
        from paper_1706_06873_b200 import dist

        r, w, dev = dist.init(backend="gloo")
        assert (r, w) == (rank, ws)
        # shard ranges cover [0, i_n) exactly once
        i_n = 32
        b, e = dist.shard(i_n, r, w)
        # K: rank 0 owns it, everybody receives it through the one broadcast
        cfg = synth.config("C1")
        K_ref = torch.from_numpy(synth.kernel_tensor(cfg, synth.KIND_GRID8, 99))
        K = K_ref.clone() if r == 0 else torch.zeros_like(K_ref)
        dist.broadcast_weights(K, 0)
        k_ok = bool(torch.equal(K, K_ref))
        # max over ranks
        m = dist.max_over_ranks(float(10 + r), dev)
        s = dist.sum_over_ranks(float(e - b), dev)
        # each rank computes its images with the oracle; the union equals the 1-process result
        small = dict(i_h=9, i_w=10, i_c=3, k_h=3, k_w=3, k_c=4)
        I_r = synth.input_images(small, b, e - b, synth.KIND_GRID8, 5)
        K_s = synth.kernel_tensor(small, synth.KIND_GRID8, 5)
        O_r = oracle.direct_conv(I_r, K_s, 1, 1)
        dist.barrier()
        q.put((r, b, e, k_ok, m, s, O_r))
        dist.finalize()
    except Exception as ex:  # noqa: BLE001
        q.put((rank, "error", repr(ex)))


def test_two_rank_gloo_driver():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    res = sorted(res, key=lambda t: t[0])
    for r in res:
        assert r[1] != "error", r
    (_, b0, e0, k0, m0, s0, O0), (_, b1, e1, k1, m1, s1, O1) = res
    assert (b0, e0, b1, e1) == (0, 16, 16, 32)
    assert k0 and k1
    assert m0 == m1 == 11.0
    assert s0 == s1 == 32.0
    import oracle
    import synth

    small = dict(i_h=9, i_w=10, i_c=3, k_h=3, k_w=3, k_c=4)
    I = synth.input_images(small, 0, 32, synth.KIND_GRID8, 5)
    O = oracle.direct_conv(I, synth.kernel_tensor(small, synth.KIND_GRID8, 5), 1, 1)
    np.testing.assert_array_equal(np.concatenate([O0, O1]), O)


@pytest.mark.parametrize("i_n,ws", [(32, 1), (32, 2), (32, 4), (32, 8), (256, 8), (1024, 8), (7, 3)])
def test_shard_partition(i_n, ws):
    from paper_1706_06873_b200 import dist

    ranges = [dist.shard(i_n, r, ws) for r in range(ws)]
    assert ranges[0][0] == 0 and ranges[-1][1] == i_n
    for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
        assert e0 == b1 and e0 >= b0
    sizes = [e - b for b, e in ranges]
    assert max(sizes) - min(sizes) <= 1


def _bench_worker(rank, ws, port, q, scaling, batch):
    """A rank of bench.py's sharding path, end to end on CPU: bench.rank_work
    picks the rank's global images, the rank generates exactly those with the
    global-index generator (bench.py's index_offset) and convolves them with
    the oracle (standing in for the device call), K comes from the one broadcast,
    the rank time is max-reduced as bench.py does."""
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(ws), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import bench
        import oracle
        import synth
        from paper_1706_06873_b200 import dist

        r, w, dev = dist.init(backend="gloo")
        rw = bench.rank_work(batch, r, w, scaling)
        small = dict(i_h=9, i_w=10, i_c=3, k_h=3, k_w=3, k_c=4)
        per = small["i_h"] * small["i_w"] * small["i_c"]
        I = synth.tensor((rw["n_local"], 9, 10, 3), 5, synth.TENSOR_I, synth.KIND_GRID8,
                         index_offset=rw["n0"] * per)
        K_ref = torch.from_numpy(synth.kernel_tensor(small, synth.KIND_GRID8, 5))
        K = K_ref.clone() if r == 0 else torch.zeros_like(K_ref)
        dist.broadcast_weights(K, 0)
        O = oracle.direct_conv(I, K.numpy(), 1, 1)
        t = dist.max_over_ranks(float(rw["n_local"]), dev)
        q.put((r, rw, O, t))
        dist.finalize()
    except Exception as ex:  # noqa: BLE001
        q.put((rank, "error", repr(ex), None))


@pytest.mark.parametrize("scaling,batch", [("strong", 6), ("strong", 7), ("weak", 3)])
def test_bench_sharding_two_ranks(scaling, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bench_worker, args=(r, 2, port, q, scaling, batch)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(2)], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    (_, rw0, O0, t0), (_, rw1, O1, t1) = res
    total = batch if scaling == "strong" else 2 * batch
    assert rw0["global_batch"] == rw1["global_batch"] == total
    assert rw0["n0"] == 0 and rw1["n0"] == rw0["n_local"] and rw0["n_local"] + rw1["n_local"] == total
    assert t0 == t1 == max(rw0["n_local"], rw1["n_local"])
    import oracle
    import synth

    small = dict(i_h=9, i_w=10, i_c=3, k_h=3, k_w=3, k_c=4)
    I = synth.input_images(small, 0, total, synth.KIND_GRID8, 5)
    O = oracle.direct_conv(I, synth.kernel_tensor(small, synth.KIND_GRID8, 5), 1, 1)
    np.testing.assert_array_equal(np.concatenate([O0, O1]), O)


def test_bench_cpu_sample_plan():
    import bench

    p = bench.cpu_sample_plan(2.0, 16, 64)  # 2 s per image on one core, 16 cores
    assert p["images"] == 8 and p["threads"] == 8 and p["est_run_s"] == 2.0 and p["runs"] == 10
    p = bench.cpu_sample_plan(5.0, 16, 64)  # 10 runs of both functions would exceed 60 s
    assert p["images"] == 4 and p["runs"] == 3
    p = bench.cpu_sample_plan(0.01, 16, 32)
    assert p["images"] == 32 and p["runs"] == 10
    p = bench.cpu_sample_plan(0.5, 8, 1)
    assert p["images"] == 1 and p["threads"] == 1
