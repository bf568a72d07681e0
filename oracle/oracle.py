"""TEST INFRASTRUCTURE — ctypes binding to the CPU oracle (liblsnif_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
leg may import this module, and only as the checker or the timed CPU
reference. The product path (paper_2504_21627_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PARITY_LIB = os.path.join(HERE, "liblsnif_oracle.so")
FAST_LIB = os.path.join(HERE, "_native", "liblsnif_oracle_fast.so")

RAY_DTYPE = np.dtype([("o", "<f4", 3), ("d", "<f4", 3), ("t_min", "<f4"), ("t_max", "<f4")])
HIT_DTYPE = np.dtype([("flags_material", "<u4"), ("t_world", "<f4"), ("normal", "<f4", 3),
                      ("albedo", "<f4", 3)])
SCENE_HIT_DTYPE = np.dtype([("t", "<f4"), ("position", "<f4", 3), ("normal", "<f4", 3),
                            ("albedo", "<f4", 3), ("kind", "<u4"), ("roughness", "<f4"),
                            ("object_index", "<i4"), ("flags", "<u4"), ("pad", "<u4", 2)])
assert RAY_DTYPE.itemsize == 32 and HIT_DTYPE.itemsize == 32 and SCENE_HIT_DTYPE.itemsize == 64

_P = C.c_void_p


def build(fast: bool = False) -> str:
    target = "fast" if fast else "all"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)
    return FAST_LIB if fast else PARITY_LIB


def _load(path: str) -> C.CDLL:
    lib = C.CDLL(path)
    f = lib
    f.oracle_last_error.restype = C.c_char_p
    f.oracle_mix_bits.restype = C.c_uint64
    f.oracle_mix_bits.argtypes = [C.c_uint64]
    f.oracle_seed_stream.restype = C.c_uint32
    f.oracle_seed_stream.argtypes = [C.c_uint64] * 4
    f.oracle_float_to_half.restype = C.c_uint16
    f.oracle_float_to_half.argtypes = [C.c_float]
    f.oracle_half_to_float.restype = C.c_float
    f.oracle_half_to_float.argtypes = [C.c_uint16]
    f.oracle_hash_vertex.restype = C.c_uint32
    f.oracle_hash_vertex.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32]
    f.oracle_ray_aabb.argtypes = [_P, _P, _P]
    f.oracle_inflate_frame.argtypes = [_P, _P]
    f.oracle_voxelize.argtypes = [_P, C.c_int, _P, C.c_int, _P, C.c_int, _P]
    f.oracle_dda_local.argtypes = [_P, _P, C.c_float, C.c_float, _P, C.c_int, C.c_int, _P, _P,
                                   _P, _P]
    f.oracle_model_load.restype = _P
    f.oracle_model_load.argtypes = [C.c_char_p]
    f.oracle_model_free.argtypes = [_P]
    f.oracle_model_save.argtypes = [_P, C.c_char_p]
    f.oracle_model_info.argtypes = [_P, _P]
    f.oracle_model_aabb.argtypes = [_P, _P]
    f.oracle_model_occupancy.restype = _P
    f.oracle_model_occupancy.argtypes = [_P]
    f.oracle_model_random.restype = _P
    f.oracle_model_random.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.c_uint32,
                                      C.c_int, C.c_int, _P, C.c_uint64]
    f.oracle_build_obj_model.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_char_p]
    f.oracle_encode_point.argtypes = [_P, C.c_int, _P, C.c_int, _P, _P, _P, _P]
    f.oracle_mlp_logits.argtypes = [_P, _P, _P]
    f.oracle_infer_batch.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, C.c_int64, _P]
    f.oracle_narrow_phase.argtypes = [_P, _P, C.c_int64, C.c_int, _P, C.c_int]
    f.oracle_time_narrow_phase.restype = C.c_double
    f.oracle_time_narrow_phase.argtypes = [_P, _P, C.c_int64, C.c_int, _P, C.c_int, C.c_int]
    f.oracle_trace.argtypes = [_P, _P, C.c_int64] + [_P] * 7
    f.oracle_build_shape_model.argtypes = [C.c_int, C.c_uint64, C.c_char_p]
    f.oracle_scene_query.argtypes = [_P, _P, C.c_int, _P, C.c_int64, C.c_int, _P, C.c_int]
    f.oracle_render.argtypes = [_P, _P, C.c_int, _P, _P, C.c_int, _P, _P, C.c_int, _P]
    f.oracle_render_debug_paths.argtypes = [_P, C.c_int64, C.c_int64, _P, _P, C.c_int]
    f.oracle_shape_mesh.argtypes = [C.c_int, _P, _P, _P, _P]
    f.oracle_label_rays.argtypes = [_P, _P, _P, _P, _P, C.c_int, _P, _P, _P, C.c_int64, _P, _P]
    f.oracle_train_batch_grad.argtypes = [_P, _P, _P, C.c_int64, _P, _P, _P]
    return lib


_LIBS: dict[str, C.CDLL] = {}


def lib(fast: bool = False) -> C.CDLL:
    path = FAST_LIB if fast else PARITY_LIB
    if path not in _LIBS:
        if not os.path.exists(path):
            build(fast)
        _LIBS[path] = _load(path)
    return _LIBS[path]


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _check(st: int, L: C.CDLL) -> None:
    if st == -1:
        raise ValueError(L.oracle_last_error().decode())
    if st < 0:
        raise RuntimeError(L.oracle_last_error().decode())


class OracleModel:
    """A loaded LSNIF model inside the oracle (model_io.cpp:116-175)."""

    def __init__(self, handle: int, fast: bool = False):
        if not handle:
            raise RuntimeError(lib(fast).oracle_last_error().decode())
        self.h = handle
        self.L = lib(fast)
        info = np.zeros(9, np.int64)
        self.L.oracle_model_info(self.h, _ptr(info))
        (self.V, self.H, self.n_levels, self.F, self.M, self.hidden, self.n_mat,
         *lv) = [int(v) for v in info]
        self.level_res = lv[: self.n_levels]
        self.aabb = np.zeros(6, np.float32)
        self.L.oracle_model_aabb(self.h, _ptr(self.aabb))

    @classmethod
    def load(cls, path: str, fast: bool = False) -> "OracleModel":
        return cls(lib(fast).oracle_model_load(path.encode()), fast)

    @classmethod
    def random(cls, occ: np.ndarray, V: int, H: int, levels, F: int, M: int, hidden: int,
               n_mat: int, frame, seed: int) -> "OracleModel":
        occ = np.ascontiguousarray(occ, np.uint8)
        lv = np.ascontiguousarray(levels, np.int32)
        fr = np.ascontiguousarray(frame, np.float32)
        L = lib()
        return cls(L.oracle_model_random(_ptr(occ), V, H, len(lv), _ptr(lv), F, M, hidden, n_mat,
                                         _ptr(fr), seed))

    def save(self, path: str) -> None:
        _check(self.L.oracle_model_save(self.h, path.encode()), self.L)

    @property
    def input_width(self) -> int:
        return self.H * self.n_levels * self.F

    def occupancy(self) -> np.ndarray:
        n = self.V ** 3 // 8
        return np.ctypeslib.as_array(C.cast(self.L.oracle_model_occupancy(self.h),
                                            C.POINTER(C.c_uint8)), (n,)).copy()

    def narrow_phase(self, rays: np.ndarray, mode: int = 0, workers: int = 0) -> np.ndarray:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        out = np.zeros(len(rays), HIT_DTYPE)
        _check(self.L.oracle_narrow_phase(self.h, _ptr(rays), len(rays), mode, _ptr(out), workers),
               self.L)
        return out

    def time_narrow_phase(self, rays: np.ndarray, mode: int = 0, workers: int = 0,
                          reps: int = 3) -> float:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        out = np.zeros(len(rays), HIT_DTYPE)
        t = self.L.oracle_time_narrow_phase(self.h, _ptr(rays), len(rays), mode, _ptr(out),
                                            workers, reps)
        if t < 0:
            _check(int(t), self.L)
        return t

    def trace(self, rays: np.ndarray) -> dict:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        n, H, Lv, F = len(rays), self.H, self.n_levels, self.F
        out = dict(info=np.zeros(n, np.int32), interval=np.zeros((n, 2), np.float32),
                   t=np.zeros((n, H), np.float32), pts=np.zeros((n, H, 3), np.float32),
                   cells=np.zeros((n, H), np.uint32), hidx=np.zeros((n, H, Lv, 8), np.uint32),
                   feat=np.zeros((n, H * Lv * F), np.float32))
        _check(self.L.oracle_trace(self.h, _ptr(rays), n, *[_ptr(out[k]) for k in
                                   ("info", "interval", "t", "pts", "cells", "hidx", "feat")]),
               self.L)
        return out

    def encode_point(self, level: int, p, volume: bool):
        p = np.ascontiguousarray(p, np.float32)
        feat = np.zeros(self.F, np.float32)
        idx = np.zeros(8, np.uint32)
        w = np.zeros(8, np.float32)
        axis = C.c_int(0)
        cnt = self.L.oracle_encode_point(self.h, level, _ptr(p), int(volume), _ptr(feat),
                                         _ptr(idx), _ptr(w), C.addressof(axis))
        return feat, idx[:cnt], w[:cnt], axis.value

    def mlp_logits(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        z = np.zeros(8 + self.n_mat, np.float32)
        self.L.oracle_mlp_logits(self.h, _ptr(x), _ptr(z))
        return z

    def infer_batch(self, inputs: np.ndarray, intervals: np.ndarray) -> np.ndarray:
        """inputs: (n, input_width) — row j is column j of the reference's MatX."""
        x = np.ascontiguousarray(inputs, np.float32)
        iv = np.ascontiguousarray(intervals, np.float32).reshape(-1, 2)
        out = np.zeros(len(x), HIT_DTYPE)
        _check(self.L.oracle_infer_batch(self.h, _ptr(x), x.shape[1] if x.ndim == 2 else 0,
                                         len(x), _ptr(iv), len(iv), _ptr(out)), self.L)
        return out

    def __del__(self):
        try:
            self.L.oracle_model_free(self.h)
        except Exception:
            pass


def build_obj_model(obj_path: str, out_path: str, V: int = 32, H: int = 18, seed: int = 0) -> None:
    L = lib()
    _check(L.oracle_build_obj_model(obj_path.encode(), V, H, seed, out_path.encode()), L)


def scene_query(models, w2o, rays: np.ndarray, mode: int = 0, workers: int = 0) -> np.ndarray:
    """Multi-object query (collect_pairs + per-object narrow phase + accept,
    renderer.cpp:154-323) over instances (models[k], w2o[k] 3x4)."""
    L = models[0].L
    rays = np.ascontiguousarray(rays, RAY_DTYPE)
    handles = (C.c_void_p * len(models))(*[m.h for m in models])
    w = np.ascontiguousarray(np.asarray(w2o, np.float32).reshape(len(models), 12))
    out = np.zeros(len(rays), SCENE_HIT_DTYPE)
    _check(L.oracle_scene_query(C.cast(handles, C.c_void_p), _ptr(w), len(models), _ptr(rays),
                                len(rays), mode, _ptr(out), workers), L)
    return out


def build_shape_model(shape: int, seed: int, out_path: str) -> None:
    L = lib()
    _check(L.oracle_build_shape_model(shape, seed, out_path.encode()), L)


def dda_local(o, d, t_min, t_max, occ: np.ndarray, res: int, cap: int):
    L = lib()
    o = np.ascontiguousarray(o, np.float32)
    d = np.ascontiguousarray(d, np.float32)
    occ = np.ascontiguousarray(occ, np.uint8)
    pts = np.zeros((max(cap, 1), 3), np.float32)
    t = np.zeros(max(cap, 1), np.float32)
    cells = np.zeros((max(cap, 1), 3), np.int32)
    fio = C.c_int(0)
    n = L.oracle_dda_local(_ptr(o), _ptr(d), t_min, t_max, _ptr(occ), res, cap, _ptr(pts),
                           _ptr(t), _ptr(cells), C.addressof(fio))
    _check(min(n, 0), L)
    return pts[:n], t[:n], cells[:n], bool(fio.value)


def ray_aabb(ray, box):
    L = lib()
    r = np.zeros(1, RAY_DTYPE)
    r["o"], r["d"], r["t_min"], r["t_max"] = ray
    b = np.ascontiguousarray(box, np.float32)
    out = np.zeros(2, np.float32)
    ok = L.oracle_ray_aabb(_ptr(r), _ptr(b), _ptr(out))
    return (float(out[0]), float(out[1])) if ok else None


def voxelize(verts: np.ndarray, faces: np.ndarray, frame, res: int) -> np.ndarray:
    L = lib()
    v = np.ascontiguousarray(verts, np.float32)
    f = np.ascontiguousarray(faces, np.int32)
    fr = np.ascontiguousarray(frame, np.float32)
    out = np.zeros(res ** 3 // 8, np.uint8)
    _check(L.oracle_voxelize(_ptr(v), len(v), _ptr(f), len(f), _ptr(fr), res, _ptr(out)), L)
    return out


# ---- path tracer (renderer.cpp:330-542), LSNIF-only scenes, primary = lsnif

def render_setup_array(camera: dict, cfg: dict, environment=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Packs RenderConfig + camera + environment into the oracle's float block."""
    a = np.zeros(20, np.float32)
    u = a.view(np.uint32)
    u[0], u[1], u[2], u[3] = cfg["width"], cfg["height"], cfg["spp"], cfg["max_bounces"]
    seed = int(cfg.get("seed", 0))
    u[4], u[5] = seed & 0xFFFFFFFF, seed >> 32
    a[6] = cfg.get("neural_eps_scale", 1e-3)
    a[7:10], a[10:13], a[13:16] = camera["position"], camera["look_at"], camera["up"]
    a[16] = camera["vfov_deg"]
    a[17:20] = environment
    return a


def lights_array(lights) -> np.ndarray:
    a = np.zeros((max(len(lights), 1), 8), np.float32)
    for i, L in enumerate(lights):
        a[i, 0:1].view(np.uint32)[0] = 1 if L["type"] == "sphere" else 0
        a[i, 1:4] = L["position"]
        a[i, 4] = L.get("radius", 0.0)
        a[i, 5:8] = L["radiance"]
    return a


def render(models, w2o, camera: dict, lights, environment, cfg: dict, world_diag,
           workers: int = 0, stats: dict | None = None) -> np.ndarray:
    """render() for instances (models[k], w2o[k]); returns (H, W, 3) float32.
    `stats` receives the intersect_scene / occluded_batch ray counts."""
    L = models[0].L
    handles = (C.c_void_p * len(models))(*[m.h for m in models])
    w = np.ascontiguousarray(np.asarray(w2o, np.float32).reshape(len(models), 12))
    setup = render_setup_array(camera, cfg, environment)
    la = lights_array(lights)
    diag = np.ascontiguousarray(world_diag, np.float32)
    img = np.zeros((cfg["height"], cfg["width"], 3), np.float32)
    st = np.zeros(2, np.int64)
    _check(L.oracle_render(C.cast(handles, C.c_void_p), _ptr(w), len(models), _ptr(setup), _ptr(la),
                           len(lights), _ptr(diag), _ptr(img), workers, _ptr(st)), L)
    if stats is not None:
        stats.update(closest_rays=int(st[0]), shadow_rays=int(st[1]))
    return img


def render_debug_paths(camera: dict, cfg: dict, first: int, n: int, k: int):
    """Primary rays and the next k uniforms of paths [first, first + n)."""
    L = lib()
    setup = render_setup_array(camera, cfg)
    rays = np.zeros(n, RAY_DTYPE)
    u = np.zeros((n, max(k, 1)), np.float32)
    _check(L.oracle_render_debug_paths(_ptr(setup), first, n, _ptr(rays), _ptr(u), k), L)
    return rays, u[:, :k]


# ---- training (training.cpp, loss.hpp, mlp.hpp backward / Adam)

TARGET_DTYPE = np.dtype([("occluded", "<i4"), ("local_t", "<f4"), ("normal", "<f4", 3),
                         ("albedo", "<f4", 3), ("material", "<i4")])
assert TARGET_DTYPE.itemsize == 36


def shape_mesh(shape: int):
    """(verts (nv, 3) f32, faces (nf, 3) i32) of a procedural fixture (shapes.cpp)."""
    L = lib()
    nv, nf = C.c_int(), C.c_int()
    _check(L.oracle_shape_mesh(shape, None, C.byref(nv), None, C.byref(nf)), L)
    v = np.zeros((nv.value, 3), np.float32)
    f = np.zeros((nf.value, 3), np.int32)
    _check(L.oracle_shape_mesh(shape, _ptr(v), C.byref(nv), _ptr(f), C.byref(nf)), L)
    return v, f


def label_rays(mesh: dict, frame, rays: np.ndarray):
    """label_ray (training.cpp:47-72) per ray -> (targets, ok)."""
    L = lib()
    rays = np.ascontiguousarray(rays, RAY_DTYPE)
    out = np.zeros(len(rays), TARGET_DTYPE)
    ok = np.zeros(len(rays), np.int8)
    arr = lambda k, t: (np.ascontiguousarray(mesh[k], t) if mesh.get(k) is not None else None)
    v, nrm, f, fn, fm = (arr("verts", np.float32), arr("normals", np.float32), arr("faces", np.int32),
                         arr("face_normals", np.int32), arr("face_material", np.int32))
    alb = np.ascontiguousarray(mesh["albedo"], np.float32)
    fr = np.ascontiguousarray(frame, np.float32)
    p = lambda a: None if a is None else _ptr(a)
    _check(L.oracle_label_rays(p(v), p(nrm), p(f), p(fn), p(fm), len(f), _ptr(alb), _ptr(fr), _ptr(rays),
                               len(rays), _ptr(out), _ptr(ok)), L)
    return out, ok


def train_batch_grad(model, rays: np.ndarray, targets: np.ndarray):
    """(loss[6], grad_mlp, grad_tables) of one batch (training.cpp:161-189)."""
    L = model.L
    rays = np.ascontiguousarray(rays, RAY_DTYPE)
    targets = np.ascontiguousarray(targets, TARGET_DTYPE)
    K1 = model.H * model.n_levels * model.F
    hid, n_out = model.hidden, 8 + model.n_mat
    n_mlp = hid * K1 + hid + hid * hid + hid + n_out * hid + n_out
    g_mlp = np.zeros(n_mlp, np.float32)
    g_tab = np.zeros(model.n_levels * model.M * model.F, np.float32)
    loss = np.zeros(6, np.float32)
    _check(L.oracle_train_batch_grad(model.h, _ptr(rays), _ptr(targets), len(rays), _ptr(loss), _ptr(g_mlp),
                                     _ptr(g_tab)), L)
    return loss, g_mlp, g_tab
