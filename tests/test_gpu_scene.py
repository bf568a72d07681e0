"""GPU parity of the multi-object path: 8
instances of 4 models under 3x4 world_to_object transforms; broad phase,
per-object narrow phase in object order, closest-hit / any-hit merge,
against the oracle's restatement of collect_pairs + run_narrow_phase +
the accept rules (renderer.cpp:154-323)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def scenes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O
    gm = [lsnif.GpuModel(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS]
    om = [O.OracleModel.load(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS]
    w2o = W.c4_world_to_object()
    gs = lsnif.GpuScene([(gm[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
    return gs, [om[k] for k in W.C4_INSTANCES], w2o, O


@pytest.mark.parametrize("which,mode", [("camera", 0), ("incoherent", 0), ("incoherent", 1)])
def test_scene_parity(scenes, which, mode):
    gs, om, w2o, O = scenes
    rays = (W.camera_rays(480, 270, camera=W.C4_CAMERA) if which == "camera"
            else W.incoherent_rays(40000, W.c4_bounds(), seed=4))
    ref = O.scene_query(om, w2o, rays, mode, 0)
    got = lsnif.scene_hits_to_numpy(gs.query(lsnif.rays_to_tensor(rays), mode))
    agree_flag = np.mean(got["flags"] == ref["flags"])
    agree_obj = np.mean(got["object_index"] == ref["object_index"])
    assert agree_flag >= 0.999 and agree_obj >= 0.999, (agree_flag, agree_obj)
    assert (ref["flags"] == 1).sum() > 100
    if mode == 0:
        both = (got["flags"] == 1) & (ref["flags"] == 1) & (got["object_index"] == ref["object_index"])
        # t tolerance: 2e-3 of the object's frame-box interval, bounded by its world diagonal
        assert np.all(np.abs(got["t"][both] - ref["t"][both]) <= 2e-3 * 4.0)
        assert np.all(np.linalg.norm(got["position"][both] - ref["position"][both], axis=1) <= 1e-2)
        cosang = np.sum(got["normal"][both] * ref["normal"][both], axis=1)
        # the face-the-ray flip (renderer.cpp:291) is discontinuous where the
        # normal is perpendicular to the ray: allow the flipped twin there
        ndotd = np.abs(np.sum(ref["normal"][both] * rays["d"][both], axis=1))
        c1 = np.cos(np.deg2rad(1.0))
        ok = (cosang >= c1) | ((ndotd < 0.02) & (np.abs(cosang) >= c1))
        assert np.all(ok), (np.sum(~ok), cosang[~ok][:5], ndotd[~ok][:5])
        assert np.all(np.abs(got["albedo"][both] - ref["albedo"][both]) <= 2e-3)
        assert np.array_equal(got["kind"][both], ref["kind"][both])
        assert np.array_equal(got["roughness"][both], ref["roughness"][both])
        miss = ref["flags"] == 0
        assert np.array_equal(got["t"][miss], rays["t_max"][miss])  # best_t untouched


def test_scene_single_instance_matches_query(scenes):
    """One identity instance == the single-object query's accepted hits."""
    gs, om, w2o, O = scenes
    m = lsnif.GpuModel(os.path.join(GOLD, "teapot_seed0.lsnif"))
    eye = np.zeros((3, 4), np.float32)
    eye[:, :3] = np.eye(3)
    s1 = lsnif.GpuScene([(m, eye)])
    rays = W.camera_rays(256, 256)
    t = lsnif.rays_to_tensor(rays)
    sh = lsnif.scene_hits_to_numpy(s1.query(t, 0))
    h = lsnif.hits_to_numpy(m.query(t, 0))
    acc = (h["flags_material"] & 4) != 0
    assert np.array_equal(sh["flags"] == 1, acc)
    assert np.array_equal(sh["t"][acc], h["t_world"][acc])
    assert np.array_equal(sh["albedo"][acc], h["albedo"][acc])


@pytest.mark.parametrize("n,mode", [(1, 0), (70001, 0), (300000, 1)])
def test_scene_query_host_matches_device(scenes, n, mode):
    """lsnif_scene_query_host (chunked H2D / scene query / D2H over the
    staging slots) returns the device path's records bit for bit, for one
    chunk and for several (ragged last chunk), pageable and pinned buffers."""
    gs = scenes[0]
    rays = W.incoherent_rays(n, W.c4_bounds(), seed=7 + n)
    dev = gs.query(lsnif.rays_to_tensor(rays), mode).cpu().numpy()
    got = gs.query_host(rays, mode)
    assert np.array_equal(got.view(np.int32).reshape(-1, 16), dev)
    pin = torch.from_numpy(rays.view(np.float32).reshape(-1, 8).copy()).pin_memory()
    out = torch.empty((n, 16), dtype=torch.int32).pin_memory()
    gs.query_host(pin, mode, out=out)
    assert np.array_equal(out.numpy(), dev)


def test_scene_more_instances_than_side_streams(scenes):
    """11 instances (more than the 8 side streams; instance k on stream k % 8)
    and an empty scene: the merged hits follow the oracle's object-order rules."""
    gs, om, w2o, O = scenes
    gm = [lsnif.GpuModel(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS]
    oms = [O.OracleModel.load(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS]
    n_inst = 11
    idx = [k % len(gm) for k in range(n_inst)]
    xf = []
    for k in range(n_inst):  # identity rotation, instances spread on a line with overlap
        m = np.zeros((3, 4), np.float32)
        m[:, :3] = np.eye(3)
        m[:, 3] = -np.array([1.3 * k - 6.5, 0.2 * (k % 3), 0.0], np.float32)
        xf.append(m)
    scene = lsnif.GpuScene([(gm[idx[k]], xf[k]) for k in range(n_inst)])
    box = np.array([-8.0, -2.0, -2.0, 8.0, 2.0, 2.0], np.float32)
    rays = W.incoherent_rays(30000, box, seed=41)
    for mode in (0, 1):
        ref = O.scene_query([oms[i] for i in idx], xf, rays, mode, 0)
        got = lsnif.scene_hits_to_numpy(scene.query(lsnif.rays_to_tensor(rays), mode))
        assert np.mean(got["flags"] == ref["flags"]) >= 0.999
        assert np.mean(got["object_index"] == ref["object_index"]) >= 0.999
        assert (ref["flags"] == 1).sum() > 100
    empty = lsnif.GpuScene([])
    e = lsnif.scene_hits_to_numpy(empty.query(lsnif.rays_to_tensor(rays[:100]), 0))
    assert np.all(e["flags"] == 0) and np.all(e["object_index"] == -1)
    assert np.array_equal(e["t"], rays["t_max"][:100])
