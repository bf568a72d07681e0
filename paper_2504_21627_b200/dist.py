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


def gather_to_rank0(local, group=None, out=None, sizes=None):
    """Gathers per-rank result tensors (first dim = rays, possibly unequal)
    into rank 0 in rank order; returns the concatenation on rank 0, None
    elsewhere. Point-to-point: every rank sends its band straight into its
    slice of rank 0's output (one batched isend / irecv set, NCCL or gloo),
    so no rank receives the other bands and nothing is re-concatenated.
    `sizes` (per-rank row counts, e.g. from row_band) skips the size
    exchange; `out` (rank 0, shape (sum(sizes),) + local.shape[1:]) is
    filled in place, so a caller that preallocates it keeps allocations out
    of its timed loop. Ranks with zero rows post no operation (every rank
    with rows joins the same single batch_isend_irecv; a communicator's
    first P2P call should therefore come from a batch in which all ranks
    take part — callers with empty bands warm up with a full batch first)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if sizes is None:
        n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
        gathered = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(gathered, n, group=group)
        sizes = [int(x.item()) for x in gathered]
    if len(sizes) != world or local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank}: {local.shape[0]} local rows but sizes = {sizes}")
    if rank != 0:
        if sizes[rank]:
            dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), 0, group)])[0].wait()
        return None
    if out is None:
        out = torch.empty((sum(sizes),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    elif out.shape != (sum(sizes),) + tuple(local.shape[1:]) or out.dtype != local.dtype:
        raise ValueError("out must hold sum(sizes) rows of local's dtype and row shape")
    offs = [0]
    for x in sizes:
        offs.append(offs[-1] + x)
    out[offs[0]:offs[1]].copy_(local)
    ops = [dist.P2POp(dist.irecv, out[offs[r]:offs[r + 1]], r, group) for r in range(1, world) if sizes[r]]
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    return out


def piece_range(band: int, pieces: int, k: int) -> tuple[int, int]:
    """Rows [s, e) of piece k when a band of `band` rows is computed in
    `pieces` consecutive pieces (the unit of compute / gather overlap)."""
    return row_band(band, pieces, k)


def gather_piece_to_rank0(local_piece, k: int, pieces: int, sizes, out=None, group=None):
    """Piece k of every rank's band into rank 0's full-frame `out` (rows in
    rank order; rank r's band starts at sum(sizes[:r])). Rank 0 computes its
    own band in place inside `out`, so only ranks 1.. transfer: each sends its
    piece k point-to-point into its slice of rank 0's output (one batched
    isend / irecv set per piece). Called by every rank for k = 0 .. pieces-1
    in order, typically on a communication stream right after piece k's
    compute, so the transfer of piece k overlaps the compute of piece k + 1
    (SURVEY.md §8(e)). Returns the async work handles (empty when this rank
    has nothing to move)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if len(sizes) != world:
        raise ValueError(f"sizes has {len(sizes)} entries for world size {world}")
    if rank != 0:
        s, e = piece_range(sizes[rank], pieces, k)
        if local_piece.shape[0] != e - s:
            raise ValueError(f"rank {rank} piece {k}: {local_piece.shape[0]} rows, expected {e - s}")
        if e == s:
            return []
        return dist.batch_isend_irecv([dist.P2POp(dist.isend, local_piece, 0, group)])
    if out is None or out.shape[0] != sum(sizes):
        raise ValueError("rank 0 needs the full-frame output (sum(sizes) rows)")
    off, ops = sizes[0], []
    for r in range(1, world):
        s, e = piece_range(sizes[r], pieces, k)
        if e > s:
            ops.append(dist.P2POp(dist.irecv, out[off + s:off + e], r, group))
        off += sizes[r]
    return dist.batch_isend_irecv(ops) if ops else []
