"""world_size-2 gloo test of the multi-GPU host path: each rank answers its
row band of a camera frame (here with the CPU oracle standing in for the GPU
kernels, which this container lacks) and the results are gathered to rank 0
with the same gather the bench uses (point-to-point into rank 0's output,
with and without known sizes / a preallocated output); the gathered frame
must equal the single-process frame bit for bit."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W_, H_ = 48, 37


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2504_21627_b200 import dist as D, workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = O.OracleModel.load(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
    rays = W.camera_rays(W_, H_, rows=D.row_band(H_, world, rank))
    hits = m.narrow_phase(rays, 0, 1)
    t = torch.from_numpy(hits.view(np.int32).reshape(-1, 8).copy())
    full = D.gather_to_rank0(t)
    # the bench's form: sizes known from the partition, output preallocated on rank 0
    sizes = [(lambda b: (b[1] - b[0]) * W_)(D.row_band(H_, world, r)) for r in range(world)]
    pre = torch.full((sum(sizes), 8), -7, dtype=torch.int32) if rank == 0 else None
    again = D.gather_to_rank0(t, out=pre, sizes=sizes)
    if rank == 0:
        assert again is pre and torch.equal(again, full)
        np.save(out_path, full.numpy())
    else:
        assert full is None and again is None
    dist.barrier()
    dist.destroy_process_group()


def _piece_worker(rank, world, port, out_path, total, pieces):
    """The bench's C5 form: each rank's band in `pieces` pieces, piece k of
    every rank gathered into rank 0's full frame right after it is computed
    (rank 0's own band written in place)."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_2504_21627_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bands = [D.ray_range(total, world, r) for r in range(world)]
    sizes = [e - s for s, e in bands]
    s0, band = bands[rank][0], sizes[rank]
    frame = torch.full((total, 4), -1, dtype=torch.int32) if rank == 0 else None
    local = frame[:band] if rank == 0 else torch.empty((band, 4), dtype=torch.int32)
    for k in range(pieces):
        ps, pe = D.piece_range(band, pieces, k)
        # "compute": a record that names its global ray index
        local[ps:pe] = torch.arange(s0 + ps, s0 + pe, dtype=torch.int32).reshape(-1, 1) * 4 + \
            torch.arange(4, dtype=torch.int32)
        for w in D.gather_piece_to_rank0(local[ps:pe], k, pieces, sizes, out=frame):
            w.wait()
    if rank == 0:
        np.save(out_path, frame.numpy())
    else:
        import pytest
        with pytest.raises(ValueError):  # a piece of the wrong length is refused, not sent
            D.gather_piece_to_rank0(local[:1], 0, pieces, sizes) if band > 1 else (_ for _ in ()).throw(ValueError())
    dist.barrier()
    dist.destroy_process_group()


def test_piecewise_band_gather(tmp_path):
    for world, total, pieces in ((2, 1001, 3), (3, 257, 8)):
        out = str(tmp_path / f"frame_{world}.npy")
        mp.spawn(_piece_worker, args=(world, _free_port(), out, total, pieces), nprocs=world, join=True)
        got = np.load(out)
        ref = np.arange(total * 4, dtype=np.int32).reshape(total, 4)
        assert np.array_equal(got, ref)


def test_row_band_sharding_and_gather(tmp_path):
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from oracle import oracle as O
    from paper_2504_21627_b200 import workloads as W
    m = O.OracleModel.load(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
    ref = m.narrow_phase(W.camera_rays(W_, H_), 0, 1).view(np.int32).reshape(-1, 8)
    got = np.load(out)
    assert got.shape == ref.shape and np.array_equal(got, ref)
