"""Multi-GPU data parallelism for the MACT path: one process per GPU.

Every pixel is independent (fast.py:86-203, lut.py:231-246), so the path
shards with NO collective on the data path: images (configs 4/5) or
contiguous cube ranges (configs 2/3) are partitioned by rank in index order.
The only exchange is the end-of-run combine of the per-GPU error partials
{sum, max, count, argmax (global index), nan} — a few dozen bytes per GPU —
all-gathered (NCCL on GPUs, gloo on CPU) and folded in rank order on every
rank, which reproduces the single-GPU statistics exactly (earliest argmax
wins ties, as harness.py:104-108 does across chunks).
"""

from __future__ import annotations

import os
from typing import List, Sequence


def env_world():
    """(rank, world, local_rank) from torchrun's environment (defaults: 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl", share_device: bool = False):
    """Initialise torch.distributed when launched by torchrun with WORLD_SIZE > 1.

    Returns (rank, world, device index).  One process per GPU: rank r drives
    cuda:LOCAL_RANK over NCCL, and a world larger than the visible device
    count is an error.  ``share_device`` (test mode for a 1-GPU box) puts
    every rank on cuda:0 and combines over gloo instead; the ranks' kernels
    never wait on one another (the path has no data-path collective).
    """
    import torch
    import torch.distributed as dist

    rank, world, local = env_world()
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if share_device:
        backend, local = "gloo", 0
    elif backend == "nccl" and local >= ndev:
        raise RuntimeError(f"rank {rank}: LOCAL_RANK {local} needs cuda:{local} but only {ndev} "
                           f"GPU(s) are visible; one process per GPU (use --share-gpu to run "
                           f"{world} ranks on cuda:0 as a host-logic test)")
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator init in the log: N ranks
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            if ndev:
                torch.cuda.set_device(local)
            dist.init_process_group(backend)
    elif ndev and backend in ("nccl", "gloo"):
        torch.cuda.set_device(local)
    return rank, world, local


def collective_device(device):
    """Device for collective tensors: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_backend() != "nccl":
        return None
    return device


def shard_range(n: int, world: int, rank: int) -> range:
    """Contiguous block partition of [0, n) (rank order = index order)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


_FIELDS = ("sum", "max", "count", "argmax", "nan")


def pack(parts: Sequence[dict]):
    """Partials -> float64 tensor (k, 5); integer fields are exact below 2^53."""
    import torch

    return torch.tensor([[float(p[f]) for f in _FIELDS] for p in parts], dtype=torch.float64)


def unpack(t) -> List[dict]:
    rows = t.tolist()
    return [{"sum": r[0], "max": r[1], "count": int(r[2]), "argmax": int(r[3]), "nan": int(r[4])}
            for r in rows]


def all_gather_partials(parts: Sequence[dict], device=None) -> List[List[dict]]:
    """All ranks' partial lists, in rank order (identity without a process group)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [list(parts)]
    t = pack(parts)
    if device is not None:
        t = t.to(device)
    bufs = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, t)
    return [unpack(b.cpu()) for b in bufs]


def combine(per_rank: Sequence[Sequence[dict]]) -> List[dict]:
    """Fold per-rank partial lists component-wise in rank order."""
    from .harness import combine_partials

    k = len(per_rank[0])
    return [combine_partials([r[c] for r in per_rank]) for c in range(k)]


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(device=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index if hasattr(device, "index") else int(device)])
        else:
            dist.barrier()
