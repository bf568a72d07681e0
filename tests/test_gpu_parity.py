"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same rays and the same model file. Gates:
  * bit-exact: pair flag, interval, DDA points / t / cells, hash indices,
    fp32 features (lsnif_debug_traverse vs oracle trace);
  * infer_batch fp32 kernel vs oracle: within 1e-5 relative;
  * full query (tcgen05 fp16 MLP): visibility and material agree on >= 99.9%
    of MLP rays; for rays both call occluded |dt| <= 2e-3*(exit-enter),
    normal angle <= 1 deg, |d albedo| <= 2e-3.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402
from helpers import edge_rays  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gmodel(teapot_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return lsnif.GpuModel(teapot_path, 0)


def workload_sets(box):
    return {
        "c1_camera_256": W.camera_rays(256, 256),
        "c3_incoherent_64k": W.incoherent_rays(65536, box, seed=3),
        "edges": edge_rays(box),
    }


@pytest.mark.parametrize("name", ["c1_camera_256", "c3_incoherent_64k", "edges"])
def test_traverse_bit_exact(gmodel, oracle_teapot, name):
    rays = workload_sets(gmodel.aabb)[name]
    ref = oracle_teapot.trace(rays)
    got = {k: v.cpu().numpy() for k, v in gmodel.debug_traverse(lsnif.rays_to_tensor(rays)).items()}
    assert np.array_equal(got["info"], ref["info"]), "pair / count / first_is_origin"
    for k in ("interval", "t", "pts", "feat"):
        assert np.array_equal(got[k].view(np.uint32), ref[k].view(np.uint32)), k
    assert np.array_equal(got["cells"].view(np.uint32), ref["cells"]), "cells"
    assert np.array_equal(got["hidx"].view(np.uint32), ref["hidx"]), "hash indices"
    assert (ref["info"] & 255).sum() > 0


def _infer_inputs(oracle_teapot, box, n=8192, seed=11):
    rays = W.incoherent_rays(n, box, seed=seed)
    tr = oracle_teapot.trace(rays)
    keep = (tr["info"] >> 9) & 1 == 1
    return tr["feat"][keep], tr["interval"][keep]


def test_infer_batch_fp32(gmodel, oracle_teapot):
    """lsnif_infer_batch_f32: fp32 in the reference's summation order, 1e-5."""
    x, iv = _infer_inputs(oracle_teapot, gmodel.aabb)
    ref = oracle_teapot.infer_batch(x, iv)
    got = lsnif.hits_to_numpy(gmodel.infer_batch(torch.from_numpy(x).cuda(),
                                                  torch.from_numpy(iv).cuda(), exact=True))
    assert np.array_equal(got["flags_material"], ref["flags_material"])
    for k in ("t_world", "normal", "albedo"):
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-5, atol=1e-6)
    with pytest.raises(ValueError):
        gmodel.infer_batch(torch.from_numpy(x).cuda(), torch.from_numpy(iv[:-1]).cuda(), exact=True)


def test_infer_batch_tcgen05(gmodel, oracle_teapot):
    """lsnif_infer_batch on the tcgen05 MLP: SURVEY App. B tolerances against
    the oracle (visibility / material >= 99.9%; for rays both call occluded
    |dt| <= 2e-3 (exit - enter), normal <= 1 degree, albedo <= 2e-3); no
    PAIR / ACCEPTED flags, as the fp32 form."""
    x, iv = _infer_inputs(oracle_teapot, gmodel.aabb, n=1 << 16, seed=12)
    ref = oracle_teapot.infer_batch(x, iv)
    got = lsnif.hits_to_numpy(gmodel.infer_batch(torch.from_numpy(x).cuda(), torch.from_numpy(iv).cuda()))
    fg, fr = got["flags_material"], ref["flags_material"]
    assert not np.any(fg & 5)
    assert np.mean((fg & 2) == (fr & 2)) >= 0.999
    assert np.mean((fg >> 8) == (fr >> 8)) >= 0.999
    both = ((fg & 2) != 0) & ((fr & 2) != 0)
    span = np.maximum(iv[:, 1] - iv[:, 0], 1e-30)
    assert np.all(np.abs(got["t_world"] - ref["t_world"])[both] <= 2e-3 * span[both] + 1e-6)
    nz = both & (np.linalg.norm(ref["normal"], axis=1) > 0)
    cosang = np.clip(np.sum(got["normal"][nz] * ref["normal"][nz], axis=1), -1.0, 1.0)
    # the sweep's rule (tests/test_gpu_full_sweep.py): near-zero normal logit
    # vectors amplify the fp16 rounding in direction
    assert np.mean(cosang >= np.cos(np.radians(1.0))) >= 0.999
    assert np.all(cosang >= np.cos(np.radians(10.0)))
    assert np.all(np.abs(got["albedo"] - ref["albedo"])[both] <= 2e-3)
    with pytest.raises(ValueError):
        gmodel.infer_batch(torch.from_numpy(x).cuda(), torch.from_numpy(iv[:-1]).cuda())


def test_infer_batch_out_of_range_inputs_use_fp32(gmodel, oracle_teapot):
    """Columns beyond the encoder range (not table interpolations) are answered
    by the fp32 kernel, decided on the device: bit-equal to the exact form."""
    x, iv = _infer_inputs(oracle_teapot, gmodel.aabb, n=4096, seed=13)
    x = x * np.float32(1e6)
    xs, ivs = torch.from_numpy(x).cuda(), torch.from_numpy(iv).cuda()
    got = lsnif.hits_to_numpy(gmodel.infer_batch(xs, ivs))
    ref = lsnif.hits_to_numpy(gmodel.infer_batch(xs, ivs, exact=True))
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def compare_query(got, ref, label):
    fg, fr = got["flags_material"], ref["flags_material"]
    assert np.array_equal(fg & 1, fr & 1), f"{label}: pair flags"
    pair = (fr & 1) == 1
    occ_g, occ_r = (fg & 2) != 0, (fr & 2) != 0
    n = max(1, pair.sum())
    vis_agree = 1 - np.sum(occ_g[pair] != occ_r[pair]) / n
    mat_agree = 1 - np.sum((fg >> 8)[pair] != (fr >> 8)[pair]) / n
    both = pair & occ_g & occ_r
    dt = np.abs(got["t_world"] - ref["t_world"])
    return vis_agree, mat_agree, both, dt


@pytest.mark.parametrize("name,mode", [("c1_camera_256", 0), ("c3_incoherent_64k", 0),
                                       ("c3_incoherent_64k", 1), ("edges", 0)])
def test_query_parity(gmodel, oracle_teapot, teapot_path, name, mode):
    rays = workload_sets(gmodel.aabb)[name]
    ref = oracle_teapot.narrow_phase(rays, mode, 0)
    got = lsnif.hits_to_numpy(gmodel.query(lsnif.rays_to_tensor(rays), mode))
    tr = oracle_teapot.trace(rays)
    span = tr["interval"][:, 1] - tr["interval"][:, 0]
    vis, mat, both, dt = compare_query(got, ref, name)
    assert vis >= 0.999 and mat >= 0.999, (vis, mat)
    assert np.all(dt[both] <= 2e-3 * span[both] + 1e-6)
    cosang = np.sum(got["normal"][both] * ref["normal"][both], axis=1)
    nz = np.sum(ref["normal"][both] ** 2, axis=1) > 0
    assert np.all(cosang[nz] >= np.cos(np.deg2rad(1.0)))
    assert np.all(np.abs(got["albedo"][both] - ref["albedo"][both]) <= 2e-3)
    # rays without boundary points take the constant zero-input output
    zero = ((tr["info"] & 255) == 0) & ((tr["info"] >> 9) & 1 == 1)
    assert np.array_equal(got["flags_material"][zero], ref["flags_material"][zero])
    np.testing.assert_allclose(got["t_world"][zero], ref["t_world"][zero], rtol=1e-6)
    # accept rule consistent with the returned t_world and the ray interval
    acc = (got["flags_material"] & 4) != 0
    occ = (got["flags_material"] & 2) != 0
    tw, t0, t1 = got["t_world"], rays["t_min"], rays["t_max"]
    rule = (tw >= t0) & (tw < t1) if mode == 0 else (tw >= t0) & (tw <= t1)
    assert np.array_equal(acc, occ & ((got["flags_material"] & 1) == 1) & rule)


def test_query_host_matches_device(gmodel):
    rays = W.incoherent_rays(3_000_000, gmodel.aabb, seed=5)  # > one staging chunk
    dev = lsnif.hits_to_numpy(gmodel.query(lsnif.rays_to_tensor(rays)))
    host = gmodel.query_host(rays)
    assert host.tobytes() == dev.tobytes()


def test_query_stats(gmodel, oracle_teapot):
    rays = W.camera_rays(256, 256)
    gmodel.query(lsnif.rays_to_tensor(rays))
    st = gmodel.last_stats()
    tr = oracle_teapot.trace(rays)
    cnt, pair = tr["info"] & 255, (tr["info"] >> 9) & 1
    assert st["rays"] == len(rays) and st["pairs"] == pair.sum()
    assert st["mlp_rows"] == np.sum(cnt > 0) and st["points"] == cnt.sum()
    assert st["volume_points"] == np.sum((tr["info"] >> 8) & 1)


def test_chunked_query_consistent(gmodel):
    """More rays than one trace/MLP launch pair takes (2^23 or 2^24 per
    stream workspace) span several launches: results must equal the
    per-slice results bit for bit (rays are independent)."""
    rays = W.incoherent_rays((1 << 24) + (1 << 20) + 7, gmodel.aabb, seed=9)
    t = lsnif.rays_to_tensor(rays)
    full = gmodel.query(t).cpu().numpy()
    part = torch.cat([gmodel.query(t[:1234567]), gmodel.query(t[1234567:])]).cpu().numpy()
    assert np.array_equal(full, part)


def test_bad_mode_raises(gmodel):
    rays = lsnif.rays_to_tensor(W.camera_rays(8, 8))
    with pytest.raises(ValueError):
        gmodel.query(rays, mode=7)


@pytest.mark.parametrize("hidden,n_mat", [(64, 2), (128, 5)])
def test_query_parity_other_widths(gmodel, oracle_teapot, tmp_path, hidden, n_mat):
    """The paper's low-quality LSNIF (hidden width 64) and a wider material
    head: a random-init model (make_sparse_hash_grid + make_mlp, seed 4) on
    the teapot's occupancy and frame, saved and loaded through the file
    format, queried through the same gates."""
    from oracle import oracle as O
    om = O.OracleModel.random(oracle_teapot.occupancy(), oracle_teapot.V, oracle_teapot.H,
                              oracle_teapot.level_res, oracle_teapot.F, oracle_teapot.M, hidden, n_mat,
                              oracle_teapot.aabb, 4)
    path = str(tmp_path / f"h{hidden}.lsnif")
    om.save(path)
    om = O.OracleModel.load(path)  # the binary16 values both sides use
    gm = lsnif.GpuModel(path)
    assert gm.info.hidden == hidden and gm.info.n_mat == n_mat
    for name in ("c1_camera_256", "c3_incoherent_64k"):
        rays = workload_sets(gm.aabb)[name]
        ref = om.narrow_phase(rays, 0, 0)
        got = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(rays)))
        tr = om.trace(rays)
        span = tr["interval"][:, 1] - tr["interval"][:, 0]
        vis, mat, both, dt = compare_query(got, ref, name)
        assert vis >= 0.999 and mat >= 0.999, (hidden, name, vis, mat)
        assert np.all(dt[both] <= 2e-3 * span[both] + 1e-6)


def test_query_pairs_given_intervals(gmodel, oracle_teapot):
    """lsnif_query_pairs (run_narrow_phase over given RayLsnifPairs): with the
    collect_pairs intervals (the oracle's, bit-exact with the kernel's own
    clip) the results equal lsnif_query's bit for bit; a stretched interval
    moves t_world = enter + sigmoid(z1) (exit - enter) accordingly; the
    lsnif_query_closest / lsnif_query_any entry points match both forms."""
    rays = W.camera_rays(256, 256)
    tr = oracle_teapot.trace(rays)
    pair = (tr["info"] >> 9) & 1 == 1
    pr, iv = rays[pair], np.ascontiguousarray(tr["interval"][pair])
    t_r, t_iv = lsnif.rays_to_tensor(pr), torch.from_numpy(iv).cuda()
    lib = lsnif.load_library()
    for mode in (lsnif.CLOSEST, lsnif.ANY):
        ref = gmodel.query(t_r, mode).cpu().numpy()
        got = gmodel.query_pairs(t_r, t_iv, mode).cpu().numpy()
        assert np.array_equal(got, ref)
        fn = lib.lsnif_query_closest if mode == lsnif.CLOSEST else lib.lsnif_query_any
        for ivp in (None, t_iv.data_ptr()):
            out = torch.empty_like(t_r, dtype=torch.int32)
            lsnif._check(fn(gmodel.h, t_r.data_ptr(), ivp, len(pr), out.data_ptr(), None))
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), ref)
    wide = iv.copy()
    wide[:, 1] = iv[:, 0] + 2.0 * (iv[:, 1] - iv[:, 0])
    a = lsnif.hits_to_numpy(gmodel.query_pairs(t_r, t_iv))
    b = lsnif.hits_to_numpy(gmodel.query_pairs(t_r, torch.from_numpy(wide).cuda()))
    assert np.array_equal(a["flags_material"] & 3, b["flags_material"] & 3)  # same MLP answers
    occ = (a["flags_material"] & 2) != 0
    np.testing.assert_allclose(b["t_world"][occ] - iv[occ, 0], 2.0 * (a["t_world"][occ] - iv[occ, 0]),
                               rtol=1e-4, atol=1e-5)
    with pytest.raises(ValueError):  # null intervals: INVALID_ARGUMENT
        lsnif._check(lib.lsnif_query_pairs(gmodel.h, t_r.data_ptr(), None, len(pr), 0, t_r.data_ptr(), None))


def test_non_finite_rays_do_not_disturb_others(gmodel):
    """NaN / Inf components (and zero directions) in some rays: the query
    terminates, and every other ray's result is bit-identical to a batch
    without them (no cross-ray contamination through shared tiles / rows)."""
    good = W.incoherent_rays(20000, gmodel.aabb, seed=13)
    bad = good[:512].copy()
    k = np.arange(len(bad))
    bad["d"][k % 4 == 0, 0] = np.nan
    bad["o"][k % 4 == 1, 1] = np.inf
    bad["d"][k % 4 == 2] = 0.0
    bad["t_max"][k % 4 == 3] = np.nan
    mixed = np.concatenate([good[:7000], bad, good[7000:]])
    ref = gmodel.query(lsnif.rays_to_tensor(good)).cpu().numpy()
    got = gmodel.query(lsnif.rays_to_tensor(mixed)).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(np.concatenate([got[:7000], got[7000 + len(bad):]]), ref)


def test_block_configurations_agree(gmodel):
    """A launch of >= 4 waves runs the 1024-thread / byte-per-cell stop-mask
    trace configuration, small launches the 256-thread / bit-mask one (whose
    DDA is checked bit for bit against the oracle above): same rays, same
    hits, bit for bit."""
    rays = W.incoherent_rays(700_000, gmodel.aabb, seed=17)
    t = lsnif.rays_to_tensor(rays)
    big = gmodel.query(t).cpu().numpy()
    small = torch.cat([gmodel.query(t[i:i + 87_500]) for i in range(0, len(rays), 87_500)]).cpu().numpy()
    assert np.array_equal(big, small)
    for mode in (lsnif.ANY,):
        assert np.array_equal(gmodel.query(t, mode).cpu().numpy(),
                              torch.cat([gmodel.query(t[i:i + 87_500], mode)
                                         for i in range(0, len(rays), 87_500)]).cpu().numpy())


def shell_occupancy(V: int) -> np.ndarray:
    """A thick spherical shell on a V^3 grid, packed as the model format
    stores it (cell x + V (y + V z), bit i & 7 of byte i >> 3)."""
    c = (np.arange(V) + 0.5) / V - 0.5
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    r = np.sqrt(x * x + y * y + z * z)
    bits = ((r > 0.25) & (r < 0.42)).reshape(-1).astype(np.uint8)
    return np.packbits(bits, bitorder="little")


@pytest.mark.parametrize("V,H,levels,F,M,hidden,n_mat", [
    (16, 12, [16, 48], 2, 50021, 64, 3),          # non-power-of-two M, F = 2
    (64, 10, [64, 128, 192], 4, 1 << 15, 128, 1),  # V = 64 (36 KB bit mask), three levels, F = 4
    (32, 16, [32, 64, 96, 128], 4, 1 << 16, 64, 8),  # the limits: L = 4, L F = 16, H L F = 256, n_mat = 8
])
def test_generic_configuration_parity(tmp_path, V, H, levels, F, M, hidden, n_mat):
    """The generic trace instantiation (anything but V = 32, L = 2, F = 3,
    power-of-two M): DDA points / t / cells, hash indices and fp32 features
    bit-exact against the oracle, and the full query through the same gates
    (SURVEY §8(a) A5-A9 at other model shapes)."""
    from oracle import oracle as O
    frame = np.array([-1.0, -0.5, -1.2, 1.1, 0.9, 1.0], np.float32)
    om = O.OracleModel.random(shell_occupancy(V), V, H, levels, F, M, hidden, n_mat, frame, 7)
    path = str(tmp_path / f"v{V}.lsnif")
    om.save(path)
    om = O.OracleModel.load(path)
    gm = lsnif.GpuModel(path)
    rays = np.concatenate([W.incoherent_rays(20000, gm.aabb, seed=23), edge_rays(gm.aabb)])
    ref = om.trace(rays)
    got = {k: v.cpu().numpy() for k, v in gm.debug_traverse(lsnif.rays_to_tensor(rays)).items()}
    assert np.array_equal(got["info"], ref["info"])
    for k in ("interval", "t", "pts", "feat"):
        assert np.array_equal(got[k].view(np.uint32), ref[k].view(np.uint32)), k
    assert np.array_equal(got["cells"].view(np.uint32), ref["cells"])
    assert np.array_equal(got["hidx"].view(np.uint32), ref["hidx"])
    assert (ref["info"] & 255).sum() > 1000
    q = om.narrow_phase(rays, 0, 0)
    g = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(rays)))
    span = ref["interval"][:, 1] - ref["interval"][:, 0]
    vis, mat, both, dt = compare_query(g, q, f"V{V}")
    assert vis >= 0.999 and mat >= 0.999, (vis, mat)
    assert np.all(dt[both] <= 2e-3 * span[both] + 1e-6)
    # lsnif_infer_batch (tcgen05 MLP at this hidden width / output count) on
    # the oracle's encoded columns, against the oracle's infer_batch
    keep = (ref["info"] >> 9) & 1 == 1
    x, iv = ref["feat"][keep], ref["interval"][keep]
    ri = om.infer_batch(x, iv)
    gi = lsnif.hits_to_numpy(gm.infer_batch(torch.from_numpy(x).cuda(), torch.from_numpy(iv).cuda()))
    assert np.mean((gi["flags_material"] & 2) == (ri["flags_material"] & 2)) >= 0.999
    assert np.mean((gi["flags_material"] >> 8) == (ri["flags_material"] >> 8)) >= 0.999
    bi = ((gi["flags_material"] & 2) != 0) & ((ri["flags_material"] & 2) != 0)
    si = np.maximum(iv[:, 1] - iv[:, 0], 1e-30)
    assert np.all(np.abs(gi["t_world"] - ri["t_world"])[bi] <= 2e-3 * si[bi] + 1e-6)


def test_fast_path_max_hit_cap_large_launch(tmp_path, oracle_teapot):
    """The fast trace shape (V = 32, L = 2, F = 3, power-of-two M) at the
    largest hit cap (H = 32, input width 192: the MLP's 2-stage X ring) in a
    launch big enough for the 1024-thread configuration, whose SMEM would not
    fit at this H (the launcher keeps 256-thread blocks): results equal the
    sliced (small-launch) query and the oracle's traversal."""
    from oracle import oracle as O
    om = O.OracleModel.random(oracle_teapot.occupancy(), 32, 32, oracle_teapot.level_res, 3,
                              oracle_teapot.M, 128, 2, oracle_teapot.aabb, 11)
    path = str(tmp_path / "h32.lsnif")
    om.save(path)
    om = O.OracleModel.load(path)
    gm = lsnif.GpuModel(path)
    rays = W.incoherent_rays(700_000, gm.aabb, seed=29)
    t = lsnif.rays_to_tensor(rays)
    big = gm.query(t).cpu().numpy()
    small = torch.cat([gm.query(t[i:i + 87_500]) for i in range(0, len(rays), 87_500)]).cpu().numpy()
    assert np.array_equal(big, small)
    sub = rays[:20000]
    ref = om.trace(sub)
    got = {k: v.cpu().numpy() for k, v in gm.debug_traverse(lsnif.rays_to_tensor(sub)).items()}
    assert np.array_equal(got["info"], ref["info"])
    assert np.array_equal(got["t"].view(np.uint32), ref["t"].view(np.uint32))
    assert np.array_equal(got["feat"].view(np.uint32), ref["feat"].view(np.uint32))
    q = om.narrow_phase(sub, 0, 0)
    vis, mat, both, dt = compare_query(lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(sub))), q, "H32")
    assert vis >= 0.999 and mat >= 0.999, (vis, mat)


@pytest.mark.parametrize("n", [0, 1, 31, 33, 127, 129, (1 << 21) - 1, (1 << 21) + 1, (1 << 23) + 1,
                               (1 << 24) + 1])
def test_batch_and_chunk_boundaries(gmodel, oracle_teapot, n):
    """Ray counts at the edges of 32-ray warp batches, 128-row MLP tiles,
    2^21-ray host staging steps and 2^23 / 2^24-ray launch chunks (and the empty
    query): every result equals the
    same rays answered inside a larger batch, bit for bit, and the pair /
    visibility flags equal the oracle's on a sample."""
    pool = W.incoherent_rays(max(n, 1) + 1000, gmodel.aabb, seed=31)
    rays = pool[1000:1000 + n]
    t_all = lsnif.rays_to_tensor(pool)
    ref = gmodel.query(t_all).cpu().numpy()[1000:1000 + n]
    got = gmodel.query(lsnif.rays_to_tensor(rays) if n else t_all[:0]).cpu().numpy()
    assert got.shape == (n, 8)
    assert np.array_equal(got, ref)
    host = gmodel.query_host(rays) if n else None
    if n:
        assert host.view(np.int32).reshape(-1, 8).tobytes() == ref.tobytes()
        k = min(n, 4096)
        q = oracle_teapot.narrow_phase(rays[:k], 0, 0)
        assert np.array_equal(got[:k, 0].view(np.uint32) & 1, q["flags_material"] & 1)


def test_cpp_adapter_example_runs():
    """examples/query_cpp (the C++ adapter: Model::load, intersect,
    infer_pairs, Scene + render) runs against the in-tree library."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "query_cpp")
    if not os.path.exists(exe):
        pytest.skip("examples/query_cpp not built (make)")
    out = subprocess.run([exe, os.path.join(root, "tests", "golden", "teapot_seed0.lsnif")],
                         capture_output=True, text=True, timeout=120, cwd=root)
    assert out.returncode == 0, out.stderr
    assert "rays accepted a neural hit" in out.stdout
    assert "infer_pairs:" in out.stdout and "render 64x36x2" in out.stdout


def test_wire_query_matches_parity_layout(gmodel, oracle_teapot):
    """lsnif_query_wire / lsnif_query_host_wire: flags, material and t_world
    bit-identical to the 32 B parity records; normal / albedo within the wire
    encoding's error (< 0.01 degree, <= 0.5/1023) and hence within the App. B
    gates against the oracle."""
    rays = W.incoherent_rays(300_000, gmodel.aabb, seed=21)
    d = lsnif.rays_to_tensor(rays)
    full = lsnif.hits_to_numpy(gmodel.query(d))
    wire = gmodel.query_wire(d)
    assert tuple(wire.shape) == (len(rays), 4)
    dec = lsnif.wire_to_hits(wire)
    assert np.array_equal(dec["flags_material"], full["flags_material"])
    assert np.array_equal(dec["t_world"].view(np.uint32), full["t_world"].view(np.uint32))
    pair = (full["flags_material"] & 1) == 1
    nz = pair & (np.sum(full["normal"] ** 2, axis=1) > 0)
    a, b = dec["normal"][nz].astype(np.float64), full["normal"][nz].astype(np.float64)
    ang = np.degrees(np.arctan2(np.linalg.norm(np.cross(a, b), axis=1), np.sum(a * b, axis=1)))
    assert ang.max() < 0.01
    assert np.all(dec["normal"][pair & ~nz] == 0)
    assert np.abs(dec["albedo"][pair] - full["albedo"][pair]).max() <= 0.5 / 1023 + 1e-7
    # host entry point: the same records
    host = gmodel.query_host_wire(rays)
    assert host.tobytes() == wire.cpu().numpy().tobytes()
    # against the oracle through the wire form (App. B gates)
    ref = oracle_teapot.narrow_phase(rays[:65536], 0, 0)
    vis, mat, both, dt = compare_query(dec[:65536], ref, "wire")
    assert vis >= 0.999 and mat >= 0.999


def test_query_rejects_bad_output_buffers(gmodel):
    d = lsnif.rays_to_tensor(W.camera_rays(16, 16))
    with pytest.raises(ValueError):
        gmodel.query(d, out=torch.empty((10, 8), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        gmodel.query_wire(d, out=torch.empty((256, 8), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        gmodel.query(d[:, :6])


def test_gpu_against_reference_golden_vectors(gmodel):
    """The GPU path against vectors written by the reference itself
    (tests/golden/make_ref_vectors.py via oracle/_ref): traversal, hash
    indices and features bit-exact; query within the App. B gates."""
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_teapot_vectors.npz"))
    rays = np.ascontiguousarray(g["rays"]).view(W.RAY_DTYPE).reshape(-1)
    got = {k: v.cpu().numpy() for k, v in gmodel.debug_traverse(lsnif.rays_to_tensor(rays)).items()}
    assert np.array_equal(got["info"], g["info"])
    for k in ("interval", "t", "pts", "feat"):
        assert np.array_equal(got[k].view(np.uint32), g[k + "_bits"]), k
    assert np.array_equal(got["cells"].view(np.uint32), g["cells"])
    assert np.array_equal(got["hidx"].view(np.uint32), g["hidx"])
    for mode, key in ((0, "hits_closest"), (1, "hits_any")):
        ref = np.ascontiguousarray(g[key]).view(lsnif.HIT_DTYPE).reshape(-1)
        hits = lsnif.hits_to_numpy(gmodel.query(lsnif.rays_to_tensor(rays), mode))
        vis, mat, both, dt = compare_query(hits, ref, key)
        assert vis >= 0.999 and mat >= 0.999


def test_gpu_against_reference_library(gmodel, teapot_path):
    """Directly against the reference's own narrow phase (oracle/_ref, built in
    the build container; the library travels with the repo)."""
    from oracle import ref as R
    if not os.path.exists(R.LIBS[False]):
        pytest.skip("oracle/_ref not built")
    rm = R.RefModel(teapot_path)
    rays = W.incoherent_rays(200_000, gmodel.aabb, seed=77)
    ref = rm.narrow_phase(rays, 0, 0)
    got = lsnif.hits_to_numpy(gmodel.query(lsnif.rays_to_tensor(rays)))
    vis, mat, both, dt = compare_query(got, ref, "ref")
    assert vis >= 0.999 and mat >= 0.999
    tr = rm.trace(rays[:20000])
    gt = {k: v.cpu().numpy() for k, v in gmodel.debug_traverse(lsnif.rays_to_tensor(rays[:20000])).items()}
    assert np.array_equal(gt["hidx"].view(np.uint32), tr["hidx"])
    assert np.array_equal(gt["feat"].view(np.uint32), tr["feat"].view(np.uint32))


def test_workspace_falls_back_when_memory_tightens(teapot_path):
    """A stream whose first query picked 2^24-ray launch pairs (plenty of free
    HBM) and whose next large query no longer fits that workspace drops to
    2^23-ray launches instead of failing; results stay bit-identical to
    per-slice queries. Runs in a subprocess: it holds most of the GPU."""
    import subprocess
    import sys
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from paper_2504_21627_b200 import lsnif, workloads as W
gm = lsnif.GpuModel({teapot_path!r}, 0)
small = lsnif.rays_to_tensor(W.camera_rays(64, 64), "cuda")
gm.query(small)  # the stream's workspace: launch size picked with the GPU nearly empty
rays = lsnif.rays_to_tensor(W.incoherent_rays((1 << 24) + 5, gm.aabb, seed=5), "cuda")
side = torch.cuda.Stream()  # the reference slices on another stream (its own workspace)
side.wait_stream(torch.cuda.current_stream())
ref = torch.cat([gm.query(rays[:3_000_001], stream=side), gm.query(rays[3_000_001:], stream=side)])
torch.cuda.synchronize()
free, _ = torch.cuda.mem_get_info()
hog = torch.empty(max(0, free - (14 << 30)), dtype=torch.uint8, device="cuda")
gm.profile_read(reset=True, stream="all")
out = gm.query(rays)
torch.cuda.synchronize()
launches = gm.profile_read(reset=True, stream="all")["trace_launches"]
assert torch.equal(out, ref)
assert launches == 3, launches  # 2^23-ray launch pairs after the fallback (2 at 2^24)
print("fallback ok", free >> 30)
"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if os.environ.get("LSNIF_CHUNK_LOG2"):
        pytest.skip("launch size fixed by LSNIF_CHUNK_LOG2")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fallback ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
