"""GPU training (lsnif::train, training.cpp:95-230) against
the oracle's restatement of the training math:

* labels: the GPU sampler's rays labelled by the oracle's label_ray
  (training.cpp:47-72, closest Moller-Trumbore hit, shading normal) must give
  the same targets (bit-exact: same float operation order);
* one batch: loss terms and every gradient (MLP weights/biases and the
  hash-grid tables, after the scatter) within 1e-4 relative L2 of the oracle's
  forward_cached + composite_loss + backward + accumulate_grad_into (fp32
  both; the GEMM summation order differs);
* training: the loss falls and the exported (binary16) model answers queries
  with a higher occlusion accuracy than the starting model.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_21627_b200 import lsnif  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INIT = os.path.join(GOLD, "sphere_seed1.lsnif")


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O
    verts, faces = O.shape_mesh(0)  # make_uv_sphere(1, 32, 16): vertex normals = positions
    mesh = dict(verts=verts, normals=verts.copy(), faces=faces, face_normals=faces.copy(),
                face_material=np.zeros(len(faces), np.int32))
    om = O.OracleModel.load(INIT)
    return O, om, mesh


def targets_np(t):
    return t.cpu().numpy().view(np.uint8).reshape(-1, 36).copy().view(lsnif.TARGET_DTYPE).reshape(-1)


def test_sampler_labels_match_oracle(setup):
    O, om, mesh = setup
    tr = lsnif.Trainer(INIT, mesh, batch=1024, seed=5)
    rays, tg = tr.sample(step=3, n=4096)
    got = targets_np(tg)
    r = rays.cpu().numpy().view(O.RAY_DTYPE).reshape(-1)
    ref, ok = O.label_rays(dict(mesh, albedo=np.full(3, 0.7, np.float32)), om.aabb, r)
    assert ok.all()
    occ = got["occluded"] == ref["occluded"]
    assert occ.mean() == 1.0
    assert 0.1 < got["occluded"].mean() < 0.9  # hits and misses (convex sphere: surface rays escape)
    for f in ("local_t", "normal", "albedo", "material"):
        assert np.array_equal(got[f], ref[f]), f


def test_batch_gradients_match_oracle(setup):
    O, om, mesh = setup
    tr = lsnif.Trainer(INIT, mesh, batch=2048, seed=9)
    rays, tg = tr.sample(step=0, n=2048)
    K1 = om.H * om.n_levels * om.F
    hid, n_out = om.hidden, 8 + om.n_mat
    n_mlp = hid * K1 + hid + hid * hid + hid + n_out * hid + n_out
    n_tab = om.n_levels * om.M * om.F
    loss, g_mlp, g_tab = tr.batch_grad(rays, tg, n_mlp, n_tab)
    ref_loss, ref_mlp, ref_tab = O.train_batch_grad(om, rays.cpu().numpy().view(O.RAY_DTYPE).reshape(-1),
                                                    targets_np(tg))
    names = ["total", "occlusion_bce", "local_t_mae", "normal_cosine", "albedo_rel_l2", "material_ce"]
    for k, name in enumerate(names):
        assert abs(loss[name] - ref_loss[k]) <= 1e-4 * max(abs(ref_loss[k]), 1e-6), (name, loss[name], ref_loss[k])
    g = g_mlp.cpu().numpy()
    offs = np.cumsum([0, hid * K1, hid, hid * hid, hid, n_out * hid, n_out])
    for part, (a, b) in zip(["w1", "b1", "w2", "b2", "w3", "b3"], zip(offs[:-1], offs[1:])):
        err = np.linalg.norm(g[a:b] - ref_mlp[a:b]) / max(np.linalg.norm(ref_mlp[a:b]), 1e-30)
        assert err <= 1e-4, (part, err)
    gt = g_tab.cpu().numpy()
    err = np.linalg.norm(gt - ref_tab) / np.linalg.norm(ref_tab)
    assert err <= 1e-4, err
    assert np.array_equal(gt != 0, ref_tab != 0)  # same touched hash entries


def occlusion_accuracy(model, rays, tg) -> float:
    hits = lsnif.hits_to_numpy(model.query(rays, lsnif.CLOSEST))
    pred = (hits["flags_material"] & lsnif.OCCLUDED) != 0
    return float(np.mean(pred == (targets_np(tg)["occluded"] != 0)))


def test_training_reduces_loss_and_improves_queries(setup):
    O, om, mesh = setup
    tr = lsnif.Trainer(INIT, mesh, batch=8192, lr=0.01, seed=1)
    first = tr.step(1)["total"]
    last = tr.step(80)
    assert last["step"] == 81
    assert last["total"] < 0.6 * first, (first, last)
    rays, tg = tr.sample(step=10**6, n=65536)  # held-out draws
    before = occlusion_accuracy(lsnif.GpuModel(INIT), rays, tg)
    after = occlusion_accuracy(tr.export(), rays, tg)
    assert after > before + 0.2 and after > 0.9, (before, after)


def test_box_labels_geometric_normals(setup):
    """A mesh without vertex normals (the box fixture): geometric normals,
    ray/box edge cases; labels bit-exact against the oracle."""
    O, _, _ = setup
    verts, faces = O.shape_mesh(1)
    mesh = dict(verts=verts, faces=faces, face_material=np.zeros(len(faces), np.int32))
    init = os.path.join(GOLD, "box_seed3.lsnif")
    tr = lsnif.Trainer(init, mesh, batch=1024, seed=11)
    rays, tg = tr.sample(step=7, n=8192)
    got = targets_np(tg)
    ref, ok = O.label_rays(dict(mesh, albedo=np.full(3, 0.7, np.float32)), O.OracleModel.load(init).aabb,
                           rays.cpu().numpy().view(O.RAY_DTYPE).reshape(-1))
    assert ok.all()
    for f in ("occluded", "local_t", "normal", "albedo", "material"):
        assert np.array_equal(got[f], ref[f]), f
    occ = got["occluded"] != 0
    n = got["normal"][occ]
    assert np.allclose(np.abs(n).max(axis=1), 1.0)  # box normals are axis-aligned


@pytest.mark.parametrize("batch", [1, 999])
def test_odd_batch_sizes(setup, batch):
    """Batches that are not multiples of the warp / tile sizes: labels and the
    batch gradients still match the oracle."""
    O, om, mesh = setup
    tr = lsnif.Trainer(INIT, mesh, batch=batch, seed=13)
    rays, tg = tr.sample(step=2, n=batch)
    K1 = om.H * om.n_levels * om.F
    hid, n_out = om.hidden, 8 + om.n_mat
    n_mlp = hid * K1 + hid + hid * hid + hid + n_out * hid + n_out
    n_tab = om.n_levels * om.M * om.F
    loss, g_mlp, g_tab = tr.batch_grad(rays, tg, n_mlp, n_tab)
    ref_loss, ref_mlp, ref_tab = O.train_batch_grad(om, rays.cpu().numpy().view(O.RAY_DTYPE).reshape(-1),
                                                    targets_np(tg))
    assert abs(loss["total"] - ref_loss[0]) <= 1e-4 * max(abs(ref_loss[0]), 1e-6)
    g = g_mlp.cpu().numpy()
    assert np.linalg.norm(g - ref_mlp) <= 1e-4 * max(np.linalg.norm(ref_mlp), 1e-30)
    gt = g_tab.cpu().numpy()
    assert np.linalg.norm(gt - ref_tab) <= 1e-4 * max(np.linalg.norm(ref_tab), 1e-30)
    tr.step(2)  # the full step loop at this batch size
