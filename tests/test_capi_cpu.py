"""CPU-only checks of the product boundary: the in-tree liblsnif_gpu.so loads
without a GPU, exports every entry point include/lsnif_gpu.h declares, fails
loudly (status + message, no crash) where a GPU or a valid file is needed,
and the host-side workload generators are deterministic and shardable."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2504_21627_b200 import lsnif, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lsnif_gpu.h")).read()
    return sorted(set(re.findall(r"\b(lsnif_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = lsnif.load_library()
    syms = header_symbols()
    assert len(syms) >= 12
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_layouts_match_reference_records():
    assert lsnif.RAY_DTYPE.itemsize == 32   # lsnif::Ray
    assert lsnif.HIT_DTYPE.itemsize == 32
    assert ctypes.sizeof(lsnif.QueryStats) == 40


def test_errors_without_gpu_or_file(tmp_path):
    lib = lsnif.load_library()
    h = ctypes.c_void_p()
    st = lib.lsnif_model_load(b"/nonexistent/model.lsnif", 0, ctypes.byref(h))
    assert st == lsnif.RUNTIME_ERROR
    assert b"cannot open model file" in lib.lsnif_last_error()
    bad = tmp_path / "bad.lsnif"
    bad.write_bytes(b"NOPE" + b"\0" * 64)
    st = lib.lsnif_model_load(str(bad).encode(), 0, ctypes.byref(h))
    assert st == lsnif.RUNTIME_ERROR and b"bad magic" in lib.lsnif_last_error()
    st = lib.lsnif_query(None, None, 0, 0, None, None)
    assert st == lsnif.INVALID_ARGUMENT


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(lsnif.LsnifError):
        lsnif._lib_backup = lsnif._lib
        try:
            lsnif._lib = None
            lsnif.load_library(str(tmp_path / "nope.so"))
        finally:
            lsnif._lib = lsnif._lib_backup


def test_incoherent_generator_is_index_addressable():
    box = np.array([-1, -1, -1, 1, 1, 1], np.float32)
    full = W.incoherent_rays(1000, box, seed=3)
    part = W.incoherent_rays(300, box, seed=3, start=500)
    assert full[500:800].tobytes() == part.tobytes()
    assert np.all((full["o"] >= box[:3]) & (full["o"] <= box[3:]))
    assert np.allclose(np.linalg.norm(full["d"], axis=1), 1, atol=1e-5)


def test_camera_row_bands_tile_the_frame():
    from paper_2504_21627_b200.dist import row_band
    full = W.camera_rays(64, 37)
    parts = [W.camera_rays(64, 37, rows=row_band(37, 3, r)) for r in range(3)]
    assert np.concatenate(parts).tobytes() == full.tobytes()


def test_shadow_rays_point_at_light():
    prim = W.camera_rays(8, 8)
    hits = np.zeros(len(prim), lsnif.HIT_DTYPE)
    hits["flags_material"][::3] = 7
    hits["t_world"] = 4.0
    hits["normal"] = (0, 1, 0)
    box = np.array([-1, 0, -1, 1, 1, 1], np.float32)
    rays, owner = W.shadow_rays(prim, hits, box)
    assert len(rays) == len(owner) and np.all(owner % 3 == 0)
    p_end = rays["o"] + rays["t_max"][:, None] / (1 - 1e-4) * rays["d"]
    assert np.allclose(p_end, W.LIGHT, atol=1e-3)


def test_render_and_trainer_fail_loudly_without_gpu_work(tmp_path):
    """Argument checks of the F3/F4 entry points run before any device work."""
    lib = lsnif.load_library()
    cfg = lsnif._config(dict(width=8, height=8, spp=1, max_bounces=1))
    cam = lsnif._camera(W.RENDER_CAMERA)
    assert lib.lsnif_render(None, None, 0, ctypes.byref(cam), None, 0, None, ctypes.byref(cfg), None, None,
                            None) == lsnif.INVALID_ARGUMENT
    assert b"null scene" in lib.lsnif_last_error()
    assert lib.lsnif_scene_query_host(None, None, 4, 0, None, None) == lsnif.INVALID_ARGUMENT
    assert b"null scene" in lib.lsnif_last_error()
    bad = lsnif._config(dict(width=0, height=8, spp=1, max_bounces=1))
    assert lib.lsnif_render_debug_paths(ctypes.byref(cam), ctypes.byref(bad), 0, 4, None, None, 0,
                                        None) == lsnif.INVALID_ARGUMENT
    h = ctypes.c_void_p()
    mesh = lsnif.MeshDesc()
    tc = lsnif.TrainConfig(1024, 0.01, 0.5, 0)
    st = lib.lsnif_trainer_create_from_file(str(tmp_path / "missing.lsnif").encode(), ctypes.byref(mesh),
                                            ctypes.byref(tc), 0, ctypes.byref(h))
    assert st == lsnif.RUNTIME_ERROR and b"cannot open model file" in lib.lsnif_last_error()
    assert lib.lsnif_trainer_step(None, 1, None, None) == lsnif.INVALID_ARGUMENT


def _oct_pack(n: np.ndarray) -> np.ndarray:
    """Independent numpy statement of the octahedral snorm16 normal map."""
    n = n.astype(np.float64)
    l1 = np.abs(n).sum(axis=1, keepdims=True)
    p = n[:, :2] / l1
    neg = n[:, 2] < 0
    sgn = np.where(p >= 0, 1.0, -1.0)
    p[neg] = ((1 - np.abs(p[neg][:, ::-1])) * sgn[neg])
    q = np.rint(np.clip(p, -1, 1) * 32767).astype(np.int64) & 0xFFFF
    return (q[:, 0] | (q[:, 1] << 16)).astype(np.uint32)


def test_wire_records_decode_within_tolerance():
    """lsnif_hits_from_wire (host decode of the packed 16 B result): flags and
    t bit-identical, normals within 0.01 degree, albedo within half a unorm10 step, the
    zero-normal marker honoured (SURVEY App. B tolerances: 1 degree, 2e-3)."""
    assert lsnif.WIRE_DTYPE.itemsize == 16
    rng = np.random.default_rng(7)
    n = 20000
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:6] = [[0, 0, 1], [0, 0, -1], [1, 0, 0], [0, -1, 0], [-1, 0, 0], [0.6, -0.8, 0]]
    alb = rng.uniform(size=(n, 3)).astype(np.float32)
    w = np.zeros(n, lsnif.WIRE_DTYPE)
    w["flags_material"] = rng.integers(0, 8, n) | (rng.integers(0, 8, n) << 8)
    w["t_world"] = rng.uniform(0, 5, n).astype(np.float32)
    w["normal_oct"] = _oct_pack(nrm)
    q = np.rint(alb.astype(np.float64) * 1023).astype(np.uint32)
    w["albedo_unorm"] = q[:, 0] | (q[:, 1] << 10) | (q[:, 2] << 20)
    w["albedo_unorm"][-1] |= lsnif.WIRE_ZERO_NORMAL
    h = lsnif.wire_to_hits(w)
    assert np.array_equal(h["flags_material"], w["flags_material"])
    assert np.array_equal(h["t_world"].view(np.uint32), w["t_world"].view(np.uint32))
    got = h["normal"][:-1].astype(np.float64)
    assert np.allclose(np.linalg.norm(got, axis=1), 1.0, atol=1e-6)
    ang = np.degrees(np.arctan2(np.linalg.norm(np.cross(got, nrm[:-1]), axis=1), np.sum(got * nrm[:-1], axis=1)))
    assert ang.max() < 0.01, ang.max()
    assert np.abs(h["albedo"] - alb).max() <= 0.5 / 1023 + 1e-7
    assert np.all(h["normal"][-1] == 0)
