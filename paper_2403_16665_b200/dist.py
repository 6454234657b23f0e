"""Batch sharding across ranks — one process per GPU.

Signals are independent, so a batch of B signals is split into contiguous
shards [lo, hi), one per rank, and every rank transforms its shard with no
communication on the data path.  Collectives appear only around it:
``max_over_ranks`` turns per-rank device times into the job time (the
slowest rank), and ``gather_shards`` / ``gather_checksums`` move results to
the verifier rank after the timed region.  The same functions run over NCCL
on B200s and over gloo on CPU (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def shard_range(total: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of a batch: sizes differ by at most one, in rank order."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} of {world_size}")
    base, extra = divmod(total, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def _coll_device(device):
    """Collectives run on `device` over NCCL, on host tensors over gloo."""
    d = _dist()
    if d is not None and d.get_backend() == "gloo":
        return "cpu"
    return device


def max_over_ranks(value: float, device=None) -> float:
    """Job time = the slowest rank's time (all-reduce MAX)."""
    import torch

    d = _dist()
    if d is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """All-reduce SUM of a per-rank count."""
    import torch

    d = _dist()
    if d is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    d.all_reduce(t, op=d.ReduceOp.SUM)
    return float(t.item())


def barrier() -> None:
    d = _dist()
    if d is not None:
        d.barrier()


def gather_checksums(out, device=None) -> list:
    """Per-rank (max|X|, sum Re X) of a rank's output shard, gathered to every rank."""
    import torch

    chk = torch.tensor([float(out.abs().amax().item()) if out.numel() else 0.0,
                        float(out.real.sum().item()) if out.numel() else 0.0],
                       dtype=torch.float64, device=_coll_device(device))
    d = _dist()
    if d is None:
        return [chk.tolist()]
    parts = [torch.zeros_like(chk) for _ in range(d.get_world_size())]
    d.all_gather(parts, chk)
    return [p.tolist() for p in parts]


def gather_shards(out, total: int, device=None):
    """Concatenate every rank's (rows, M) output shard on every rank (untimed verification).

    Shards may differ by one row; they are padded to the largest shard for the
    collective and trimmed afterwards.
    """
    import torch

    d = _dist()
    if d is None:
        return out
    ws = d.get_world_size()
    sizes = [hi - lo for lo, hi in (shard_range(total, ws, r) for r in range(ws))]
    width = out.shape[1]
    buf = torch.zeros((max(sizes), width), dtype=out.dtype, device=_coll_device(out.device))
    buf[: out.shape[0]] = out
    real = torch.view_as_real(buf) if buf.is_complex() else buf
    parts = [torch.zeros_like(real) for _ in range(ws)]
    d.all_gather(parts, real)
    parts = [torch.view_as_complex(p) if buf.is_complex() else p for p in parts]
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0).to(out.device)
