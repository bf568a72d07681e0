"""Multi-GPU plumbing for the query path.

Ray queries are independent: a frame is sharded into contiguous row bands,
one per rank, with no communication during compute; each rank regenerates
its own rays from the index-addressable generators. The only collective is
the final result gather to rank 0 (NCCL over NVLink on GPUs, gloo in the CPU
tests). Output bits are identical for 1 vs N ranks because every ray is
answered by the same kernels regardless of how the frame is split.
"""
from __future__ import annotations


def row_band(height: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row band [y0, y1) of `rank` (sizes differ by at most 1)."""
    base, extra = divmod(height, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def ray_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [s, e) of an n-ray index space."""
    return row_band(n, world, rank)


def gather_to_rank0(local, group=None):
    """Gathers per-rank result tensors (first dim = rays, possibly unequal)
    into rank 0 in rank order; returns the concatenation on rank 0, None
    elsewhere. Uses all_gather of padded equal-size buffers (one collective
    for the sizes, one for the payload)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)])
