"""TEST INFRASTRUCTURE — ctypes binding to the LSNIF reference itself,
compiled from /root/reference/proj/src by oracle/Makefile.ref against the
Eigen-subset shim (oracle/_ref/libref_{parity,fast}.so, see ref_capi.cpp).

Only tests/, __graft_entry__ and bench.py's CPU arms may use it, as the
checker or the timed CPU reference. The built libraries travel to the GPU
box; they can only be (re)built where /root/reference exists.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_ROOT = "/root/reference/proj"
LIBS = {False: os.path.join(HERE, "_ref", "libref_parity.so"),
        True: os.path.join(HERE, "_ref", "libref_fast.so")}

RAY_DTYPE = np.dtype([("o", "<f4", 3), ("d", "<f4", 3), ("t_min", "<f4"), ("t_max", "<f4")])
HIT_DTYPE = np.dtype([("flags_material", "<u4"), ("t_world", "<f4"), ("normal", "<f4", 3),
                      ("albedo", "<f4", 3)])
SCENE_HIT_DTYPE = np.dtype([("t", "<f4"), ("position", "<f4", 3), ("normal", "<f4", 3),
                            ("albedo", "<f4", 3), ("kind", "<u4"), ("roughness", "<f4"),
                            ("object_index", "<i4"), ("flags", "<u4"), ("pad", "<u4", 2)])
_P = C.c_void_p


def available(fast: bool = False) -> bool:
    return os.path.exists(LIBS[fast]) or os.path.isdir(REF_ROOT)


def build() -> None:
    """Builds both libraries (needs /root/reference; a no-op when up to date)."""
    if not os.path.isdir(REF_ROOT):
        if all(os.path.exists(p) for p in LIBS.values()):
            return
        raise RuntimeError("oracle/_ref is not built and /root/reference is absent")
    subprocess.run(["make", "-s", "-C", HERE, "-f", "Makefile.ref", "all"], check=True)


_LIBS: dict[bool, C.CDLL] = {}


def lib(fast: bool = False) -> C.CDLL:
    if fast not in _LIBS:
        if not os.path.exists(LIBS[fast]) or os.path.isdir(REF_ROOT):
            build()
        L = C.CDLL(LIBS[fast])
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_load.restype = _P
        L.ref_model_load.argtypes = [C.c_char_p]
        L.ref_model_free.argtypes = [_P]
        L.ref_model_info.argtypes = [_P, _P]
        L.ref_model_aabb.argtypes = [_P, _P]
        L.ref_trace.argtypes = [_P, _P, C.c_int64] + [_P] * 7
        L.ref_infer_batch.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, C.c_int64, _P]
        L.ref_narrow_phase.argtypes = [_P, _P, C.c_int64, C.c_int, _P, C.c_int]
        L.ref_scene_query.argtypes = [_P, _P, C.c_int64, C.c_int, _P, C.c_int]
        L.ref_time_scene_query.restype = C.c_double
        L.ref_time_scene_query.argtypes = [_P, _P, C.c_int64, C.c_int, _P, C.c_int, C.c_int]
        L.ref_build_obj_model.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_uint64]
        L.ref_build_shape_model.argtypes = [C.c_int, C.c_uint64, C.c_char_p]
        _LIBS[fast] = L
    return _LIBS[fast]


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class RefModel:
    """load_model (model_io.cpp:116-175) + a one-object PreparedScene."""

    def __init__(self, path: str, fast: bool = False):
        self.L = lib(fast)
        self.h = self.L.ref_model_load(path.encode())
        if not self.h:
            raise RuntimeError(self.L.ref_last_error().decode())
        info = np.zeros(9, np.int64)
        self.L.ref_model_info(self.h, _ptr(info))
        (self.V, self.H, self.n_levels, self.F, self.M, self.hidden, self.n_mat, *lv) = [int(v) for v in info]
        self.input_width = self.H * self.n_levels * self.F
        box = np.zeros(6, np.float32)
        self.L.ref_model_aabb(self.h, _ptr(box))
        self.aabb = box

    def _check(self, st: int) -> None:
        if st == -1:
            raise ValueError(self.L.ref_last_error().decode())
        if st < 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def trace(self, rays: np.ndarray) -> dict:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        n, H, L, lf = len(rays), self.H, self.n_levels, self.n_levels * self.F
        out = dict(info=np.zeros(n, np.int32), interval=np.zeros((n, 2), np.float32),
                   t=np.zeros((n, H), np.float32), pts=np.zeros((n, H, 3), np.float32),
                   cells=np.zeros((n, H), np.uint32), hidx=np.zeros((n, H, L, 8), np.uint32),
                   feat=np.zeros((n, H * lf), np.float32))
        self._check(self.L.ref_trace(self.h, _ptr(rays), n, *[_ptr(out[k]) for k in
                                                             ("info", "interval", "t", "pts", "cells", "hidx",
                                                              "feat")]))
        return out

    def infer_batch(self, inputs: np.ndarray, intervals: np.ndarray) -> np.ndarray:
        """inputs (n, rows): row j = column j of the reference's MatX."""
        x = np.ascontiguousarray(inputs, np.float32)
        iv = np.ascontiguousarray(intervals, np.float32).reshape(-1, 2)
        out = np.zeros(x.shape[0], HIT_DTYPE)
        self._check(self.L.ref_infer_batch(self.h, _ptr(x), x.shape[1], x.shape[0], _ptr(iv), iv.shape[0],
                                           _ptr(out)))
        return out

    def narrow_phase(self, rays: np.ndarray, mode: int = 0, workers: int = 0) -> np.ndarray:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        out = np.zeros(len(rays), HIT_DTYPE)
        self._check(self.L.ref_narrow_phase(self.h, _ptr(rays), len(rays), mode, _ptr(out), workers))
        return out

    def scene_query(self, rays: np.ndarray, mode: int = 0, workers: int = 0) -> np.ndarray:
        """PreparedScene::intersect_scene (mode 0) / occluded_batch (mode 1)."""
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        out = np.zeros(len(rays), SCENE_HIT_DTYPE)
        self._check(self.L.ref_scene_query(self.h, _ptr(rays), len(rays), mode, _ptr(out), workers))
        return out

    def time_scene_query(self, rays: np.ndarray, mode: int = 0, workers: int = 0, reps: int = 3) -> float:
        rays = np.ascontiguousarray(rays, RAY_DTYPE)
        out = np.zeros(len(rays), SCENE_HIT_DTYPE)
        t = self.L.ref_time_scene_query(self.h, _ptr(rays), len(rays), mode, _ptr(out), workers, reps)
        if t < 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        return t

    def __del__(self):
        try:
            self.L.ref_model_free(self.h)
        except Exception:
            pass


def build_obj_model(obj_path: str, out_path: str, V: int = 32, H: int = 18, seed: int = 0) -> None:
    """The reference's train() setup state (T = 0) for an OBJ mesh, saved as LSNF v1."""
    L = lib(False)
    if L.ref_build_obj_model(obj_path.encode(), out_path.encode(), V, H, seed) != 0:
        raise RuntimeError(L.ref_last_error().decode())


def build_shape_model(shape: int, seed: int, out_path: str) -> None:
    """Same for a shapes.cpp fixture: 0 sphere, 1 box (1, .6, .8), 2 torus."""
    L = lib(False)
    if L.ref_build_shape_model(shape, seed, out_path.encode()) != 0:
        raise RuntimeError(L.ref_last_error().decode())


def hardware_concurrency(fast: bool = True) -> int:
    return int(lib(fast).ref_hardware_concurrency())
