"""Concurrent callers (SURVEY §8(b) Threading: render() calls intersect_scene /
occluded_batch from several worker threads on one const PreparedScene,
renderer.cpp:483; results must not depend on worker count or order,
renderer.hpp:24-26). Host threads share one model / scene and each queries on
its own CUDA stream (per-stream workspaces inside the library), or through the
host-buffer entry points; every result must equal the sequential one bit for
bit."""
import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def run_threads(fns):
    errors = []

    def wrap(fn):
        try:
            fn()
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gm = lsnif.GpuModel(os.path.join(GOLD, "teapot_seed0.lsnif"))
    sets = [W.camera_rays(192, 160), W.incoherent_rays(150000, gm.aabb, seed=21),
            W.incoherent_rays(70000, gm.aabb, seed=22), W.camera_rays(320, 200)]
    return gm, sets


def test_concurrent_device_queries(setup):
    gm, sets = setup
    ref = [[gm.query(lsnif.rays_to_tensor(r), mode).cpu().numpy() for mode in (0, 1)] for r in sets]
    got = [[None, None] for _ in sets]

    def worker(k):
        def fn():
            s = torch.cuda.Stream()
            d = lsnif.rays_to_tensor(sets[k])
            torch.cuda.current_stream().synchronize()
            with torch.cuda.stream(s):
                outs = []
                for it in range(6):
                    outs.append(gm.query(d, it % 2, stream=s))
                s.synchronize()
            got[k] = [outs[-2].cpu().numpy(), outs[-1].cpu().numpy()]
            for it, o in enumerate(outs):
                assert np.array_equal(o.cpu().numpy(), ref[k][it % 2]), (k, it)
        return fn

    run_threads([worker(k) for k in range(len(sets))])
    for k in range(len(sets)):
        for mode in (0, 1):
            assert np.array_equal(got[k][mode], ref[k][mode])


def test_concurrent_host_queries(setup):
    gm, sets = setup
    ref = [gm.query_host(r, 0) for r in sets]
    res = [None] * len(sets)

    def worker(k):
        def fn():
            for _ in range(3):
                res[k] = gm.query_host(sets[k], 0)
                assert res[k].tobytes() == ref[k].tobytes(), k
        return fn

    run_threads([worker(k) for k in range(len(sets))])


def test_concurrent_scene_queries():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    models = [lsnif.GpuModel(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS]
    w2o = W.c4_world_to_object()
    scene = lsnif.GpuScene([(models[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
    sets = [W.camera_rays(160, 90, camera=W.C4_CAMERA), W.incoherent_rays(60000, W.c4_bounds(), seed=31),
            W.incoherent_rays(90000, W.c4_bounds(), seed=32)]
    ref = [scene.query(lsnif.rays_to_tensor(r), 0).cpu().numpy() for r in sets]

    def worker(k):
        def fn():
            s = torch.cuda.Stream()
            d = lsnif.rays_to_tensor(sets[k])
            torch.cuda.current_stream().synchronize()
            with torch.cuda.stream(s):
                for _ in range(4):
                    out = scene.query(d, 0, stream=s)
                s.synchronize()
            assert np.array_equal(out.cpu().numpy(), ref[k]), k
            h = scene.query_host(sets[k], 0)
            assert np.array_equal(h.view(np.int32).reshape(-1, 16), ref[k]), k
        return fn

    run_threads([worker(k) for k in range(len(sets))])


def test_concurrent_models_of_different_shapes(setup, tmp_path):
    """Host threads querying models whose kernels need different dynamic
    SMEM (the teapot's 18-point pools and a V = 64 model's 36 KB bit mask) on
    their own streams: the per-kernel SMEM limit is only ever raised, so no
    thread's launch is invalidated by another's attribute call."""
    from oracle import oracle as O
    gm, sets = setup
    occ = np.packbits((np.random.default_rng(5).random(64 ** 3) < 0.08).astype(np.uint8), bitorder="little")
    om = O.OracleModel.random(occ, 64, 24, [64, 128], 3, 1 << 16, 128, 2,
                              np.array([-1, -1, -1, 1, 1, 1], np.float32), 3)
    path = str(tmp_path / "v64.lsnif")
    om.save(path)
    g64 = lsnif.GpuModel(path)
    models = [gm, g64]
    rays = [W.incoherent_rays(60000, m.aabb, seed=50 + k) for k, m in enumerate(models)]
    ref = [m.query(lsnif.rays_to_tensor(r)).cpu().numpy() for m, r in zip(models, rays)]

    def worker(k):
        def fn():
            s = torch.cuda.Stream()
            ds = [lsnif.rays_to_tensor(r) for r in rays]
            torch.cuda.current_stream().synchronize()
            with torch.cuda.stream(s):
                outs = [models[(k + it) % 2].query(ds[(k + it) % 2], stream=s) for it in range(8)]
                s.synchronize()
            for it, o in enumerate(outs):
                assert np.array_equal(o.cpu().numpy(), ref[(k + it) % 2]), (k, it)
        return fn

    run_threads([worker(k) for k in range(4)])
