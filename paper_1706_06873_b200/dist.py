"""Multi-GPU driver: one process per GPU, images sharded, K broadcast once.

MEC's loops run "in parallel" over the images n (Alg.2 l.4, l.17, l.22;
P:156-190) and K is the only operand every image needs, so the path shards
over i_n with no data-path collective: rank r owns the contiguous global
images [r*i_n/g, (r+1)*i_n/g) (contiguous slices of I and O in NHWC) and the
only NCCL call is one broadcast of K from rank 0 over NVLink / NVSwitch.
Timing helpers take the max over ranks (measurement only, outside the path).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None) -> tuple[int, int, torch.device]:
    """Initialise the process group if WORLD_SIZE > 1 and bind this rank's GPU."""
    rank, ws, local = world()
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    else:
        dev = torch.device("cpu")
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        be = backend or ("nccl" if dev.type == "cuda" else "gloo")
        kw = {"device_id": dev} if be == "nccl" else {}
        dist.init_process_group(be, rank=rank, world_size=ws, **kw)
    return rank, ws, dev


def shard(i_n: int, rank: int, ws: int) -> tuple[int, int]:
    """Global image range [begin, end) owned by `rank` (contiguous, balanced)."""
    return (i_n * rank) // ws, (i_n * (rank + 1)) // ws


def broadcast_weights(K: torch.Tensor, src: int = 0) -> torch.Tensor:
    """The single collective of the path: K from rank `src` to all ranks."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(K, src)
    return K


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(x: float, device: torch.device) -> float:
    """Measurement only: max of a per-rank scalar (e.g. elapsed ms)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([float(x)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return float(x)


def sum_over_ranks(x: float, device: torch.device) -> float:
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([float(x)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())
    return float(x)


def finalize() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()
