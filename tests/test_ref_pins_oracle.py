"""The oracle pinned to the REFERENCE ITSELF (CPU, no GPU).

oracle/_ref is the reference's own source tree (/root/reference/proj/src),
compiled in place against the Eigen-subset shim (oracle/Makefile.ref,
oracle/ref_capi.cpp). These tests check, bit for bit:
  * the test fixtures: the reference's train() setup state (voxelize_surface,
    make_sparse_hash_grid, make_mlp: mt19937 + libstdc++ distributions,
    binary16 save_model) reproduces every committed .lsnif fixture byte for
    byte;
  * the oracle restatement against the reference on the same rays: pair
    intervals, DDA points / t / cells, hash indices, fp32 features
    (collect_boundary_hits_local, encode_ray_into), infer_batch outputs, the
    narrow phase with both accept rules, and PreparedScene::intersect_scene /
    occluded_batch accept decisions.
Both sides are the IEEE (-ffp-contract=off) builds; the MLP products sum
the inner index in ascending order in both (Eigen's own GEMM order is
library-internal; the shim's is documented in oracle/eigen_shim/Eigen/Core).
"""
import filecmp
import os

import numpy as np
import pytest

from helpers import edge_rays
from paper_2504_21627_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
TEAPOT_OBJ = "/root/reference/proj/assets/teapot.obj"


def _ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return ref


@pytest.fixture(scope="module")
def R():
    return _ref()


@pytest.fixture(scope="module")
def ref_teapot(R, teapot_path):
    return R.RefModel(teapot_path)


def test_reference_regenerates_the_fixtures(R, tmp_path):
    for shape, seed, name in [(0, 1, "sphere_seed1"), (2, 2, "torus_seed2"), (1, 3, "box_seed3")]:
        out = str(tmp_path / f"{name}.lsnif")
        R.build_shape_model(shape, seed, out)
        assert filecmp.cmp(out, os.path.join(GOLD, name + ".lsnif"), shallow=False), name
    if os.path.exists(TEAPOT_OBJ):
        out = str(tmp_path / "teapot.lsnif")
        R.build_obj_model(TEAPOT_OBJ, out, 32, 18, 0)
        assert filecmp.cmp(out, os.path.join(GOLD, "teapot_seed0.lsnif"), shallow=False)


def ray_sets(box):
    prim = W.camera_rays(160, 90)
    return {
        "c1_camera": W.camera_rays(128, 128),
        "c3_incoherent": W.incoherent_rays(16384, box, seed=3),
        "c5_incoherent": W.incoherent_rays_at(np.arange(0, 3840 * 2160 * 16, 8101, dtype=np.uint64), box, seed=5),
        "edges": edge_rays(box),
        "camera_160": prim,
    }


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint32) if a.dtype != np.uint32 else a


@pytest.mark.parametrize("name", ["c1_camera", "c3_incoherent", "c5_incoherent", "edges"])
def test_trace_matches_reference(ref_teapot, oracle_teapot, name):
    rays = ray_sets(oracle_teapot.aabb)[name]
    a, b = oracle_teapot.trace(rays), ref_teapot.trace(rays)
    for k in ("info", "interval", "t", "pts", "cells", "hidx", "feat"):
        assert np.array_equal(_bits(a[k]), _bits(b[k])), k
    assert (a["info"] & 255).sum() > 0


@pytest.mark.parametrize("name", ["c1_camera", "c3_incoherent", "c5_incoherent", "edges"])
@pytest.mark.parametrize("mode", [0, 1])
def test_narrow_phase_matches_reference(ref_teapot, oracle_teapot, name, mode):
    rays = ray_sets(oracle_teapot.aabb)[name]
    a, b = oracle_teapot.narrow_phase(rays, mode, 0), ref_teapot.narrow_phase(rays, mode, 0)
    assert a.tobytes() == b.tobytes()


def test_infer_batch_matches_reference(ref_teapot, oracle_teapot):
    rays = W.incoherent_rays(4096, oracle_teapot.aabb, seed=41)
    tr = oracle_teapot.trace(rays)
    keep = (tr["info"] >> 9) & 1 == 1
    x, iv = tr["feat"][keep], tr["interval"][keep]
    assert oracle_teapot.infer_batch(x, iv).tobytes() == ref_teapot.infer_batch(x, iv).tobytes()
    with pytest.raises(ValueError):  # std::invalid_argument (renderer.cpp:185-189)
        ref_teapot.infer_batch(x, iv[:-1])


def test_scene_queries_match_accept_rules(ref_teapot, oracle_teapot):
    """PreparedScene::intersect_scene / occluded_batch (the reference's public
    query API) accept exactly the rays the narrow-phase records accept, with
    the same t and material albedo."""
    rays = np.concatenate([W.camera_rays(96, 96), W.incoherent_rays(8192, oracle_teapot.aabb, seed=9)])
    for mode in (0, 1):
        h = oracle_teapot.narrow_phase(rays, mode, 0)
        s = ref_teapot.scene_query(rays, mode, 0)
        acc = (h["flags_material"] & 4) != 0
        assert np.array_equal(s["flags"] == 1, acc)
        if mode == 0:
            assert np.array_equal(s["t"][acc].view(np.uint32), h["t_world"][acc].view(np.uint32))
            assert np.array_equal(s["albedo"][acc], h["albedo"][acc])


@pytest.mark.parametrize("name", ["sphere_seed1", "torus_seed2", "box_seed3"])
def test_other_fixtures_match_reference(R, name):
    from oracle import oracle as O
    path = os.path.join(GOLD, name + ".lsnif")
    om, rm = O.OracleModel.load(path), R.RefModel(path)
    rays = W.incoherent_rays(8192, om.aabb, seed=13)
    assert om.narrow_phase(rays, 0, 0).tobytes() == rm.narrow_phase(rays, 0, 0).tobytes()
    a, b = om.trace(rays), rm.trace(rays)
    assert np.array_equal(_bits(a["feat"]), _bits(b["feat"]))


def test_golden_vectors_match_reference(ref_teapot):
    """tests/golden/ref_teapot_vectors.npz (written by
    tests/golden/make_ref_vectors.py from the reference) still reproduces."""
    g = np.load(os.path.join(GOLD, "ref_teapot_vectors.npz"))
    rays = g["rays"].view(W.RAY_DTYPE).reshape(-1)
    assert ref_teapot.narrow_phase(rays, 0, 0).view(np.uint32).tobytes() == g["hits_closest"].tobytes()
    tr = ref_teapot.trace(rays)
    assert np.array_equal(tr["info"], g["info"])
    assert np.array_equal(_bits(tr["feat"]), g["feat_bits"])
