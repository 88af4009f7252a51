"""Multi-GPU plumbing for the TPO path.

Every tensor product is independent, so the batch is split into contiguous
per-rank shards and each rank runs the kernels on its own device with no
collective on the data path.  Collectives only appear after the compute:
max-reduction of per-rank device times and gathers of results / checksums
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of n_total items for `rank`; shard sizes
    differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_total < 0:
        raise ValueError("n_total must be >= 0")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, n_total: int, device=None):
    """All-gather the row-sharded tensor `local` ([rows_r, ...]) into the full
    [n_total, ...] tensor on every rank (uneven shards are padded)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    cap = shard_range(n_total, world, 0)[1]
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    out = [parts[r][: shard_range(n_total, world, r)[1] - shard_range(n_total, world, r)[0]] for r in range(world)]
    return torch.cat(out, dim=0)


def gather_checksums(values, device=None) -> list:
    """All-gather a small per-rank vector of checksums; returns one list per rank."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(values, dtype=torch.float64, device=device).reshape(-1)
    if not (dist.is_available() and dist.is_initialized()):
        return [t.cpu().tolist()]
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [p.cpu().tolist() for p in parts]
