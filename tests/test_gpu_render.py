"""GPU parity of the wavefront path tracer (render(),
renderer.cpp:330-542, PrimaryMode::lsnif, LSNIF-only scene) against the
oracle's CPU restatement.

* Sampling is bit-exact: primary rays and every uniform draw of a path's
  mt19937 stream (renderer.cpp:347-361, sampling.hpp:12-14).
* Direct lighting (max_bounces = 0: camera ray, closest neural hit, NEE to a
  point and a sphere light, shadow query): per pixel within the stated
  tolerance — the hits differ only by the MLP's fp16-vs-fp32 numerics.
* Full paths (4 bounces, diffuse + glossy): a path's direction after the
  first bounce depends on the MLP normal, so paths decorrelate and the
  comparison is statistical: the GPU-vs-oracle image error must be at the
  level of the oracle's own Monte-Carlo noise (two seeds), and the image
  means must agree.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def scene(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O
    tmp = tmp_path_factory.mktemp("render")
    paths = [os.path.join(GOLD, n + ".lsnif") for n in W.RENDER_MODELS]
    # glossy lid on the teapot, glossy sphere: exercises the Phong branch
    paths[0] = W.glossy_copy(paths[0], str(tmp / "teapot_glossy.lsnif"), 1, 0.3)
    paths[1] = W.glossy_copy(paths[1], str(tmp / "sphere_glossy.lsnif"), 0, 0.2)
    gm = [lsnif.GpuModel(p) for p in paths]
    om = [O.OracleModel.load(p) for p in paths]
    w2o = W.render_world_to_object()
    gs = lsnif.GpuScene([(gm[i], w2o[i]) for i in range(len(gm))])
    diag = W.world_diag_from_frames([m.aabb for m in om])
    return gs, om, w2o, diag, O


def both(scene, cfg, lights=None):
    gs, om, w2o, diag, O = scene
    lights = W.RENDER_LIGHTS if lights is None else lights
    got = gs.render(W.RENDER_CAMERA, lights, W.RENDER_ENV, cfg, diag).cpu().numpy()
    ref = O.render(om, w2o, W.RENDER_CAMERA, lights, W.RENDER_ENV, cfg, diag, workers=0)
    return got, ref


@pytest.mark.parametrize("seed", [0, 123456789])
def test_render_sampling_bit_exact(seed):
    from oracle import oracle as O
    cfg = dict(width=160, height=90, spp=4, max_bounces=4, seed=seed)
    n, k = 160 * 90 * 4, 40
    rays, u = lsnif.render_debug_paths(W.RENDER_CAMERA, cfg, 0, n, k)
    ref_rays, ref_u = O.render_debug_paths(W.RENDER_CAMERA, cfg, 0, n, k)
    got_rays = rays.cpu().numpy().view(np.uint32).reshape(-1, 8)
    assert np.array_equal(got_rays, ref_rays.view(np.uint32).reshape(-1, 8))
    assert np.array_equal(u.cpu().numpy().view(np.uint32), ref_u.view(np.uint32))
    # the last servable draw (index 226) of a far path
    r2, u2 = lsnif.render_debug_paths(W.RENDER_CAMERA, cfg, n - 1, 1, 225)
    _, v2 = O.render_debug_paths(W.RENDER_CAMERA, cfg, n - 1, 1, 225)
    assert np.array_equal(u2.cpu().numpy().view(np.uint32), v2.view(np.uint32))


def test_render_direct_lighting_parity(scene):
    cfg = dict(width=96, height=64, spp=2, max_bounces=0, seed=3)
    got, ref = both(scene, cfg)
    env = np.float32(W.RENDER_ENV)
    lit = ~np.all(np.isclose(ref, env, rtol=1e-6), axis=-1)
    assert lit.mean() > 0.05  # the scene is actually hit
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)
    close = np.all(rel <= 1e-2, axis=-1)
    # tolerance: 99% of pixels within 1% (relative, 1e-3 floor); the rest are
    # pixels where a visibility / shadow decision flips near the 0.5 boundary
    print(f"direct: lit {lit.mean():.3f} close {close.mean():.5f} mean {got.mean():.6f} vs {ref.mean():.6f}")
    assert close.mean() >= 0.99, close.mean()
    assert abs(got.mean() - ref.mean()) <= 5e-3 * ref.mean()


def test_render_full_paths_statistical_parity(scene):
    gs, om, w2o, diag, O = scene
    cfg = dict(width=64, height=40, spp=8, max_bounces=4, seed=11)
    got, ref = both(scene, cfg)
    ref2 = O.render(om, w2o, W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, dict(cfg, seed=12),
                    diag, workers=0)
    assert np.isfinite(got).all() and (got >= 0).all()
    noise = np.sqrt(np.mean((ref2 - ref) ** 2))
    err = np.sqrt(np.mean((got - ref) ** 2))
    close = np.mean(np.all(np.abs(got - ref) <= 1e-2 * np.maximum(np.abs(ref), 1e-3), axis=-1))
    print(f"full paths: err {err:.5f} noise {noise:.5f} close {close:.4f} "
          f"mean {got.mean():.5f} vs {ref.mean():.5f}")
    # most paths follow the oracle's exactly (same streams, hits within the
    # MLP tolerance); the error must stay well under the Monte-Carlo noise
    assert err <= 0.5 * noise, (err, noise)
    assert abs(got.mean() - ref.mean()) <= 0.03 * ref.mean(), (got.mean(), ref.mean())


def test_render_deterministic_waves_and_errors(scene):
    gs, om, w2o, diag, O = scene
    cfg = dict(width=48, height=30, spp=4, max_bounces=3, seed=5)
    a = gs.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag).cpu().numpy()
    b = gs.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV,
                  dict(cfg, max_paths_in_flight=48 * 4 * 7), diag).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))  # wave size is not semantic
    too_many = [dict(type="sphere", position=(0, 5, 0), radius=0.1, radiance=(1, 1, 1))] * 30
    with pytest.raises(lsnif.LsnifError, match="227"):
        gs.render(W.RENDER_CAMERA, too_many, W.RENDER_ENV, cfg, diag)
    with pytest.raises(ValueError, match="world_diag"):  # std::invalid_argument
        gs.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag[:-1])


def test_render_rotated_shared_instances():
    """The C4 layout (8 instances of 4 shared models, yaw 0 / 45 degrees):
    direct lighting per pixel against the oracle through rotated transforms."""
    from oracle import oracle as O
    gm = {n: lsnif.GpuModel(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS}
    om = {n: O.OracleModel.load(os.path.join(GOLD, n + ".lsnif")) for n in W.C4_MODELS}
    names = [W.C4_MODELS[k] for k in W.C4_INSTANCES]
    w2o = W.c4_world_to_object()
    gs = lsnif.GpuScene([(gm[n], w2o[i]) for i, n in enumerate(names)])
    diag = W.world_diag_from_frames([om[n].aabb for n in names])
    cam = dict(position=(0.0, 6.0, 14.0), look_at=(0.0, 0.3, 0.0), up=(0.0, 1.0, 0.0), vfov_deg=50.0)
    lights = [dict(type="point", position=(0.0, 8.0, 6.0), radiance=(60.0, 60.0, 60.0))]
    cfg = dict(width=128, height=72, spp=1, max_bounces=0, seed=2)
    got = gs.render(cam, lights, W.RENDER_ENV, cfg, diag).cpu().numpy()
    ref = O.render([om[n] for n in names], w2o, cam, lights, W.RENDER_ENV, cfg, diag, workers=0)
    lit = ~np.all(np.isclose(ref, np.float32(W.RENDER_ENV), rtol=1e-6), axis=-1)
    assert lit.mean() > 0.02
    close = np.all(np.abs(got - ref) <= 1e-2 * np.maximum(np.abs(ref), 1e-3), axis=-1)
    assert close.mean() >= 0.99, close.mean()
