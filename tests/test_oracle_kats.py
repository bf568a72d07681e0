"""Pins the CPU oracle (oracle/) against every known-answer example SPEC.md
gives for the hot path (the reference ships no tests or golden vectors;
SURVEY.md §4, §8(c)). CPU only."""
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O

INF = float("inf")


def occ_grid(V, cells):
    bits = np.zeros(V ** 3 // 8, np.uint8)
    for (x, y, z) in cells:
        i = x + V * (y + V * z)
        bits[i >> 3] |= np.uint8(1 << (i & 7))
    return bits


# ---- half.hpp codec (model_io DESIGN DECISIONS: IEEE binary16, RNE)
def test_half_codec_matches_ieee():
    L = O.lib()
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-9, 6, 20000),
                           np.array([0.0, -0.0, 1.0, 65504.0, 65520.0, 1e-8, 6.1e-5, 5.96e-8, 2.98e-8,
                                     np.inf, -np.inf], np.float32)]).astype(np.float32)
    ours = np.array([L.oracle_float_to_half(float(v)) for v in vals], np.uint16)
    ref = vals.astype(np.float16).view(np.uint16)
    assert np.array_equal(ours, ref)
    allh = np.arange(65536, dtype=np.uint16)
    f = np.array([L.oracle_half_to_float(int(h)) for h in allh], np.float32)
    ref = allh.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(f[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert np.all(np.isnan(f[nan]))


def test_seed_stream_splitmix():
    L = O.lib()
    # mix_bits(0) is the published splitmix64 first output for state 0.
    assert L.oracle_mix_bits(0) == 0xE220A8397B1DCDAF
    assert L.oracle_seed_stream(0, 0x9DD1, 0, 0) != L.oracle_seed_stream(1, 0x9DD1, 0, 0)


# ---- geometry: ray_aabb_intersect
def test_ray_aabb_kats():
    box = [0, 0, 0, 1, 1, 1]
    assert O.ray_aabb(((-2, .5, .5), (1, 0, 0), 0.0, INF), box) == (2.0, 3.0)
    assert O.ray_aabb(((.5, .5, .5), (0, 0, 1), 0.0, INF), box) == (0.0, 0.5)
    assert O.ray_aabb(((-2, 2, .5), (1, 0, 0), 0.0, INF), box) is None  # d=0 axis outside


def test_ray_aabb_marching():
    rng = np.random.default_rng(1)
    box = np.array([0, 0, 0, 1, 1, 1], np.float32)
    bad = 0
    for _ in range(2000):
        o = rng.uniform(-2, 3, 3).astype(np.float32)
        d = rng.standard_normal(3).astype(np.float32)
        d /= np.linalg.norm(d)
        r = O.ray_aabb((o, d, 0.0, INF), box)
        ts = np.arange(0, 8, 1e-3, dtype=np.float64)
        p = o[None].astype(np.float64) + ts[:, None] * d[None]
        inside = np.all((p >= -1e-9) & (p <= 1 + 1e-9), axis=1)
        if inside.any():
            t0, t1 = ts[inside][0], ts[inside][-1]
            bad += r is None or abs(r[0] - t0) > 2e-3 or abs(r[1] - t1) > 2e-3
        else:
            bad += r is not None and (r[1] - r[0]) > 2e-3
    assert bad == 0


def test_inflate_frame():
    L = O.lib()
    out = np.zeros(6, np.float32)
    box = np.array([0, 0, 0, 2, 1, 1], np.float32)
    L.oracle_inflate_frame(box.ctypes.data, out.ctypes.data)
    pad = np.float32(1e-4) * np.float32(2)
    assert np.array_equal(out, np.array([-pad, -pad, -pad, 2 + pad, 1 + pad, 1 + pad], np.float32))


# ---- voxelizer
def test_voxelize_kats():
    frame = [0, 0, 0, 1, 1, 1]
    empty = O.voxelize(np.zeros((0, 3)), np.zeros((0, 3), np.int32), frame, 32)
    assert empty.size == 4096 and empty.sum() == 0
    tri = np.array([[0.51, 0.51, 0.51], [0.52, 0.51, 0.51], [0.51, 0.52, 0.51]], np.float32)
    one = O.voxelize(tri, np.array([[0, 1, 2]], np.int32), frame, 32)
    assert int(np.unpackbits(one).sum()) == 1
    quad = np.array([[0, 0, .5], [1, 0, .5], [1, 1, .5], [0, 1, .5]], np.float32)
    g = O.voxelize(quad, np.array([[0, 1, 2], [0, 2, 3]], np.int32), frame, 4)
    # z = 0.5 lies on the iz=1/iz=2 boundary: both layers (double assignment)
    assert int(np.unpackbits(g).sum()) == 32


# ---- DDA
def test_dda_single_cell_kat():
    occ = occ_grid(4, [(0, 1, 1)])
    pts, t, cells, fio = O.dda_local((-0.1, 0.375, 0.375), (1, 0, 0), 0.0, INF, occ, 4, 18)
    assert len(pts) == 1 and not fio
    assert np.array_equal(pts[0], np.array([0, 0.375, 0.375], np.float32))
    assert tuple(cells[0]) == (0, 1, 1)
    assert abs(t[0] - 0.1) < 1e-6


def test_dda_empty_grid():
    occ = occ_grid(32, [])
    pts, *_ = O.dda_local((-0.1, 0.3, 0.2), (1, 0.1, 0.2), 0.0, INF, occ, 32, 18)
    assert len(pts) == 0


def test_dda_properties_random():
    rng = np.random.default_rng(2)
    V = 32
    for g in range(3):
        occ = (rng.random(V ** 3 // 8 * 8) < 0.15).astype(np.uint8)
        occ = np.packbits(occ, bitorder="little")
        for _ in range(300):
            o = rng.uniform(-0.5, 1.5, 3).astype(np.float32)
            d = rng.standard_normal(3).astype(np.float32)
            pts, t, cells, fio = O.dda_local(o, d, 0.0, INF, occ, V, 3 * V)
            assert np.all(np.diff(t) > 0)  # strict ordering
            for k, (p, c) in enumerate(zip(pts, cells)):
                i = c[0] + V * (c[1] + V * c[2])
                assert (occ[i >> 3] >> (i & 7)) & 1  # occupied cells only
                if k == 0 and fio:
                    continue
                on_face = np.min(np.abs(p * V - np.round(p * V))) < 1e-4
                assert on_face
            # cap property: first-H truncation of the uncapped list
            pts18, t18, c18, _ = O.dda_local(o, d, 0.0, INF, occ, V, 18)
            n = min(18, len(t))
            assert np.array_equal(t18, t[:n]) and np.array_equal(c18, cells[:n])


def test_dda_inside_origin_first_point():
    occ = occ_grid(4, [(1, 1, 1), (2, 1, 1)])
    pts, t, cells, fio = O.dda_local((0.3, 0.3, 0.3), (1, 0.01, 0.02), 0.0, INF, occ, 4, 18)
    assert fio and tuple(cells[0]) == (1, 1, 1) and t[0] == 0.0
    assert np.array_equal(pts[0], np.array([0.3, 0.3, 0.3], np.float32))
    assert len(pts) == 2 and pts[1][0] == np.float32(0.5)


def test_dda_marching_oracle():
    """Occupied-cell sequence equals a fine marcher (acceptance 3)."""
    rng = np.random.default_rng(3)
    V = 32
    occ = np.packbits((rng.random(V ** 3) < 0.1).astype(np.uint8), bitorder="little")
    bits = np.unpackbits(occ, bitorder="little")
    mism = 0
    N = 400
    for _ in range(N):
        o = rng.uniform(-0.3, 1.3, 3).astype(np.float32)
        d = rng.standard_normal(3).astype(np.float32)
        d /= np.linalg.norm(d)
        _, _, cells, _ = O.dda_local(o, d, 0.0, INF, occ, V, 3 * V)
        ts = np.arange(0, 4, 1e-4 / V * 10)
        p = o[None].astype(np.float64) + ts[:, None] * d[None]
        inside = np.all((p >= 0) & (p < 1), axis=1)
        c = np.floor(p[inside] * V).astype(int)
        seq = []
        for cc in c:
            if not seq or tuple(cc) != seq[-1]:
                seq.append(tuple(cc))
        occ_seq = [s for s in seq if bits[s[0] + V * (s[1] + V * s[2])]]
        mism += occ_seq != [tuple(x) for x in cells]
    assert mism <= N * 0.01  # boundary-tie rays only


# ---- hash + encode
def test_hash_kats():
    L = O.lib()
    M = 1 << 17
    assert L.oracle_hash_vertex(0, 0, 0, M) == 0
    assert L.oracle_hash_vertex(1, 0, 0, M) == 1
    assert L.oracle_hash_vertex(0, 1, 0, M) == 2654435761 % M
    assert L.oracle_hash_vertex(0, 0, 1, M) == 805459861 % M
    x, y, z = 37, 101, 5
    h = (x ^ ((y * 2654435761) & 0xFFFFFFFF) ^ ((z * 805459861) & 0xFFFFFFFF)) % M
    assert L.oracle_hash_vertex(x, y, z, M) == h


def test_encode_kats(oracle_teapot):
    m = oracle_teapot
    tab = [None, None]
    # at a grid vertex on a voxel plane: the vertex's own entry on each level
    p = np.array([8 / 32, 20 / 64, 40 / 128], np.float32)
    for lvl, R in enumerate(m.level_res):
        feat, idx, w, axis = m.encode_point(lvl, p, False)
        assert len(idx) == 4 and axis == 0
        k = int(np.argmax(w))
        assert w[k] == 1.0 and np.sum(w) == 1.0
    # face centre: mean of the 4 entries (weights 0.25 each)
    p = np.array([0.25, (10 + 0.5) / 64, (20 + 0.5) / 64], np.float32)
    feat, idx, w, axis = m.encode_point(0, p, False)
    assert axis == 0 and np.allclose(w, 0.25)
    # volume point: 8 corners, partition of unity
    feat, idx, w, axis = m.encode_point(1, np.array([0.3, 0.4, 0.7], np.float32), True)
    assert len(idx) == 8 and axis == -1 and abs(w.sum() - 1) < 1e-6


def test_encode_matches_dense_trilinear(oracle_teapot):
    """Boundary points: the 4-corner encoding equals dense 8-corner trilinear
    interpolation of the same hashed entries within 1e-6."""
    m = oracle_teapot
    rng = np.random.default_rng(4)
    for _ in range(200):
        p = rng.random(3).astype(np.float32)
        a = rng.integers(0, 3)
        p[a] = np.float32(rng.integers(0, 33) / 32)
        f4, idx, w, axis = m.encode_point(1, p, False)
        f8, idx8, w8, _ = m.encode_point(1, p, True)
        assert axis == a and len(idx) <= 4
        assert np.allclose(f4, f8, atol=1e-6 * 1e-4 + 1e-12, rtol=1e-5)


def test_encode_ray_zero_padding(oracle_teapot):
    from paper_2504_21627_b200 import workloads as W
    rays = W.camera_rays(64, 64)
    tr = oracle_teapot.trace(rays)
    cnt = tr["info"] & 255
    lf = oracle_teapot.n_levels * oracle_teapot.F
    for i in range(len(rays)):
        assert np.all(tr["feat"][i, cnt[i] * lf:].view(np.uint32) == 0)
    assert np.any(cnt == 0) and np.any(cnt > 0)


# ---- MLP / infer_batch
def _zero_model(n_mat):
    return O.OracleModel.random(np.zeros(512, np.uint8), 16, 18, [32, 64], 3, 1 << 10, 16,
                                n_mat, [0, 0, 0, 1, 1, 1], 0)


def test_mlp_zero_input_heads():
    m = _zero_model(3)
    out = m.infer_batch(np.zeros((1, m.input_width), np.float32), np.array([[1.0, 3.0]]))
    # random weights, zero biases, zero input: z == 0 exactly
    assert (out["flags_material"][0] & 2) == 0  # sigmoid(0) = 0.5 is not > 0.5
    assert out["t_world"][0] == 2.0               # enter + 0.5 * (exit - enter)
    assert np.all(out["normal"][0] == 0)
    assert np.all(out["albedo"][0] == 0.5)
    assert out["flags_material"][0] >> 8 == 0     # uniform softmax, first argmax


def test_infer_batch_shape_errors():
    m = _zero_model(1)
    with pytest.raises(ValueError):
        m.infer_batch(np.zeros((2, m.input_width), np.float32), np.zeros((3, 2), np.float32))
    with pytest.raises(ValueError):
        m.infer_batch(np.zeros((2, m.input_width + 1), np.float32), np.zeros((2, 2), np.float32))


def test_infer_batch_equivariance(oracle_teapot):
    from paper_2504_21627_b200 import workloads as W
    m = oracle_teapot
    rays = W.camera_rays(48, 48)
    tr = m.trace(rays)
    x, iv = tr["feat"], tr["interval"]
    out = m.infer_batch(x, iv)
    perm = np.random.default_rng(5).permutation(len(x))
    outp = m.infer_batch(x[perm], iv[perm])
    assert outp.tobytes() == out[perm].tobytes()
    one = m.infer_batch(x[7:8], iv[7:8])
    assert one.tobytes() == out[7:8].tobytes()


# ---- model file
def test_model_roundtrip_and_footprint(tmp_path, oracle_teapot, teapot_path):
    p = str(tmp_path / "rt.lsnif")
    oracle_teapot.save(p)
    assert open(p, "rb").read() == open(teapot_path, "rb").read()
    m = oracle_teapot
    n_params = 108 * 128 + 128 + 128 * 128 + 128 + 128 * 10 + 10
    assert n_params == 31754
    expected = 4 + 8 * 4 + 4096 + 2 * (4 + (1 << 17) * 3 * 2) + 2 * n_params + 4 + 2 * 20 + 24
    assert os.path.getsize(teapot_path) == expected == 1640580
    # SPEC.md:538 defaults with N_mat = 1: 4,096 / 1,572,864 / 63,250 B
    assert 32 ** 3 // 8 == 4096 and 2 * (1 << 17) * 3 * 2 == 1572864
    assert (108 * 128 + 128 + 128 * 128 + 128 + 128 * 9 + 9) * 2 == 63250


def test_model_load_errors(tmp_path, teapot_path):
    raw = open(teapot_path, "rb").read()
    bad = tmp_path / "bad.lsnif"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        O.OracleModel.load(str(bad))
    bad.write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(RuntimeError, match="version"):
        O.OracleModel.load(str(bad))
    bad.write_bytes(raw[:1000])
    with pytest.raises(RuntimeError, match="truncated"):
        O.OracleModel.load(str(bad))


def test_teapot_fixture_statistics(oracle_teapot):
    """The fixture reproduces the survey's independent probe."""
    from paper_2504_21627_b200 import workloads as W
    m = oracle_teapot
    assert int(np.unpackbits(m.occupancy()).sum()) == 3634
    tr = m.trace(W.camera_rays(128, 128))
    cnt, pair = tr["info"] & 255, (tr["info"] >> 9) & 1
    assert abs(pair.mean() - 0.656) < 0.01
    assert abs(cnt[pair == 1].mean() - 3.64) < 0.15


def test_oracle_reproduces_reference_golden_vectors(oracle_teapot):
    """The golden vectors written by the reference itself
    (tests/golden/make_ref_vectors.py, oracle/_ref) pin the restatement even
    where /root/reference is absent: DDA / hash / features and both
    narrow-phase accept rules, bit for bit."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_teapot_vectors.npz"))
    rays = np.ascontiguousarray(g["rays"]).view(oracle_teapot_ray_dtype()).reshape(-1)
    tr = oracle_teapot.trace(rays)
    assert np.array_equal(tr["info"], g["info"])
    for k in ("interval", "t", "pts", "feat"):
        assert np.array_equal(np.asarray(tr[k]).view(np.uint32), g[k + "_bits"]), k
    assert np.array_equal(tr["cells"], g["cells"]) and np.array_equal(tr["hidx"], g["hidx"])
    assert oracle_teapot.narrow_phase(rays, 0, 1).view(np.uint32).tobytes() == g["hits_closest"].tobytes()
    assert oracle_teapot.narrow_phase(rays, 1, 1).view(np.uint32).tobytes() == g["hits_any"].tobytes()


def oracle_teapot_ray_dtype():
    from oracle import oracle as O
    return O.RAY_DTYPE
