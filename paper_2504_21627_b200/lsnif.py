"""Python host mirror of the reference's LSNIF query API over the C ABI
(include/lsnif_gpu.h, liblsnif_gpu.so built in-tree for sm_100a).

Reference interface mirrored (proj/include/lsnif/renderer.hpp):
  * ``load_model(path)``                    -> model_io.hpp:45 (+ device upload)
  * ``infer_batch(model, inputs, intervals)`` -> renderer.hpp:52-53
  * ``GpuModel.intersect(rays)``             -> intersect_scene's narrow phase +
                                               closest-hit accept (renderer.cpp:269-303)
  * ``GpuModel.occluded(rays)``              -> occluded_batch (renderer.cpp:305-323)
Errors are raised as the reference's exception types: ValueError for
std::invalid_argument, RuntimeError for std::runtime_error.

There is no CPU fallback: importing a missing/unloadable extension raises.
PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSNIF_LIB") or os.path.join(HERE, "liblsnif_gpu.so")  # override: A/B builds

RAY_DTYPE = np.dtype([("o", "<f4", 3), ("d", "<f4", 3), ("t_min", "<f4"), ("t_max", "<f4")])
HIT_DTYPE = np.dtype([("flags_material", "<u4"), ("t_world", "<f4"), ("normal", "<f4", 3),
                      ("albedo", "<f4", 3)])
# lsnif_hit_wire: packed 16 B result (octahedral snorm16 normal, unorm10 albedo)
WIRE_DTYPE = np.dtype([("flags_material", "<u4"), ("t_world", "<f4"), ("normal_oct", "<u4"),
                       ("albedo_unorm", "<u4")])
WIRE_ZERO_NORMAL = 0x40000000
SCENE_HIT_DTYPE = np.dtype([("t", "<f4"), ("position", "<f4", 3), ("normal", "<f4", 3),
                            ("albedo", "<f4", 3), ("kind", "<u4"), ("roughness", "<f4"),
                            ("object_index", "<i4"), ("flags", "<u4"), ("pad", "<u4", 2)])
PAIR, OCCLUDED, ACCEPTED = 1, 2, 4
CLOSEST, ANY = 0, 1

OK, INVALID_ARGUMENT, RUNTIME_ERROR, CUDA_ERROR, UNSUPPORTED = range(5)


class LsnifError(RuntimeError):
    pass


class ModelInfo(C.Structure):
    _fields_ = [("voxel_res", C.c_int32), ("hit_cap", C.c_int32), ("n_levels", C.c_int32),
                ("f_dim", C.c_int32), ("table_size", C.c_uint32), ("hidden", C.c_int32),
                ("n_mat", C.c_int32), ("n_materials", C.c_int32), ("level_res", C.c_int32 * 4),
                ("aabb", C.c_float * 6), ("activation_scale", C.c_float),
                ("device_bytes", C.c_uint64), ("device", C.c_int32)]


class Profile(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("trace_launches", C.c_uint64),
                ("mlp_launches", C.c_uint64), ("trace_ms", C.c_double), ("mlp_ms", C.c_double)]


class QueryStats(C.Structure):
    _fields_ = [("rays", C.c_int64), ("pairs", C.c_int64), ("mlp_rows", C.c_int64),
                ("points", C.c_int64), ("volume_points", C.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads liblsnif_gpu.so; raises if it is missing (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LsnifError(f"liblsnif_gpu.so not built at {path}; run `make` "
                         "(or __graft_entry__.build())")
    lib = C.CDLL(path)
    P = C.c_void_p
    lib.lsnif_last_error.restype = C.c_char_p
    lib.lsnif_build_info.restype = C.c_char_p
    lib.lsnif_model_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(P)]
    lib.lsnif_model_destroy.argtypes = [P]
    lib.lsnif_model_get_info.argtypes = [P, C.POINTER(ModelInfo)]
    lib.lsnif_query.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_query_host.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_query_wire.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_query_host_wire.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_hits_from_wire.argtypes = [P, C.c_int64, P]
    lib.lsnif_query_pairs.argtypes = [P, P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_query_closest.argtypes = [P, P, P, C.c_int64, P, P]
    lib.lsnif_query_any.argtypes = [P, P, P, C.c_int64, P, P]
    lib.lsnif_infer_batch.argtypes = [P, P, C.c_int64, C.c_int64, P, C.c_int64, P, P]
    lib.lsnif_infer_batch_f32.argtypes = [P, P, C.c_int64, C.c_int64, P, C.c_int64, P, P]
    lib.lsnif_debug_traverse.argtypes = [P, P, C.c_int64] + [P] * 7 + [P]
    lib.lsnif_last_query_stats.argtypes = [P, P, C.POINTER(QueryStats)]
    lib.lsnif_profile_enable.argtypes = [P, C.c_int]
    lib.lsnif_scene_create.argtypes = [P, C.c_int32, C.POINTER(P)]
    lib.lsnif_scene_destroy.argtypes = [P]
    lib.lsnif_scene_query.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_scene_query_host.argtypes = [P, P, C.c_int64, C.c_int, P, P]
    lib.lsnif_profile_read.argtypes = [P, P, C.c_int, C.POINTER(Profile)]
    lib.lsnif_render.argtypes = [P, P, C.c_int32, P, P, C.c_int32, P, P, P, P, P]
    lib.lsnif_render_debug_paths.argtypes = [P, P, C.c_int64, C.c_int64, P, P, C.c_int32, P]
    lib.lsnif_trainer_create_from_file.argtypes = [C.c_char_p, P, P, C.c_int, C.POINTER(P)]
    lib.lsnif_trainer_destroy.argtypes = [P]
    lib.lsnif_trainer_step.argtypes = [P, C.c_int32, P, P]
    lib.lsnif_trainer_export.argtypes = [P, C.POINTER(P)]
    lib.lsnif_trainer_batch_grad.argtypes = [P, P, P, C.c_int64, P, P, P, P]
    lib.lsnif_trainer_sample.argtypes = [P, C.c_int64, C.c_int64, P, P, P]
    for name in ("lsnif_model_load", "lsnif_model_destroy", "lsnif_model_get_info", "lsnif_query",
                 "lsnif_query_host", "lsnif_query_wire", "lsnif_query_host_wire",
                 "lsnif_hits_from_wire", "lsnif_query_pairs", "lsnif_query_closest", "lsnif_query_any",
                 "lsnif_infer_batch", "lsnif_infer_batch_f32", "lsnif_debug_traverse",
                 "lsnif_last_query_stats", "lsnif_profile_enable", "lsnif_profile_read",
                 "lsnif_scene_create", "lsnif_scene_destroy", "lsnif_scene_query",
                 "lsnif_scene_query_host", "lsnif_render",
                 "lsnif_render_debug_paths", "lsnif_trainer_create_from_file", "lsnif_trainer_destroy",
                 "lsnif_trainer_step", "lsnif_trainer_export", "lsnif_trainer_batch_grad",
                 "lsnif_trainer_sample"):
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _check(st: int) -> None:
    if st == OK:
        return
    msg = load_library().lsnif_last_error().decode()
    if st == INVALID_ARGUMENT:
        raise ValueError(msg)
    raise LsnifError(f"lsnif status {st}: {msg}")


def _torch():
    import torch
    return torch


def _check_rays(rays):
    """Query input: a contiguous (n, 8) float32 CUDA tensor (lsnif_ray records).
    No implicit copy: a temporary could be freed before an asynchronous
    launch on another stream reads it."""
    torch = _torch()
    if not (rays.is_cuda and rays.dtype == torch.float32 and rays.dim() == 2 and rays.shape[1] == 8):
        raise ValueError("rays must be an (n, 8) float32 CUDA tensor")
    if not rays.is_contiguous():
        raise ValueError("rays must be contiguous")
    return rays


def _check_out(out, shape, device):
    """Query output: allocated when None, else an int32 contiguous tensor of
    `shape` on `device` (an undersized buffer would be written out of bounds)."""
    torch = _torch()
    if out is None:
        return torch.empty(shape, dtype=torch.int32, device=device)
    if out.dtype != torch.int32 or tuple(out.shape) != tuple(shape) or out.device != device \
            or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous int32 tensor of shape {tuple(shape)} on {device}")
    return out


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class GpuModel:
    """A device-resident LSNIF model (one per object; shareable across instances)."""

    def __init__(self, path: str, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        _check(lib.lsnif_model_load(path.encode(), device, C.byref(h)))
        self.h = h
        self.device = device
        info = ModelInfo()
        _check(lib.lsnif_model_get_info(self.h, C.byref(info)))
        self.info = info
        self.H, self.n_levels, self.F = info.hit_cap, info.n_levels, info.f_dim
        self.input_width = self.H * self.n_levels * self.F
        self.aabb = np.array(list(info.aabb), np.float32)

    def close(self):
        if getattr(self, "h", None):
            load_library().lsnif_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- device API (torch CUDA tensors) ----
    def query(self, rays, mode: int = CLOSEST, out=None, stream=None):
        """rays: CUDA tensor (n, 8) float32 (lsnif_ray records). Returns (n, 8)
        int32 tensor of lsnif_hit records (view with hits_to_numpy)."""
        rays = _check_rays(rays)
        n = rays.shape[0]
        out = _check_out(out, (n, 8), rays.device)
        _check(load_library().lsnif_query(self.h, rays.data_ptr(), n, mode, out.data_ptr(),
                                          _stream_ptr(stream)))
        return out

    def query_wire(self, rays, mode: int = CLOSEST, out=None, stream=None):
        """lsnif_query_wire: (n, 4) int32 tensor of packed 16 B lsnif_hit_wire
        records (wire_to_hits expands them)."""
        torch = _torch()
        rays = _check_rays(rays)
        n = rays.shape[0]
        out = _check_out(out, (n, 4), rays.device)
        _check(load_library().lsnif_query_wire(self.h, rays.data_ptr(), n, mode, out.data_ptr(),
                                               _stream_ptr(stream)))
        return out

    def query_pairs(self, rays, intervals, mode: int = CLOSEST, out=None, stream=None):
        """run_narrow_phase (renderer.cpp:232-265): every ray is a pair with the
        given [t_enter, t_exit] (CUDA tensor (n, 2) float32) instead of the
        in-kernel frame clip. Returns (n, 8) int32 lsnif_hit records."""
        torch = _torch()
        rays = _check_rays(rays)
        if not (intervals.is_cuda and intervals.dtype == torch.float32 and intervals.is_contiguous()
                and tuple(intervals.shape) == (rays.shape[0], 2) and intervals.device == rays.device):
            raise ValueError("intervals must be a contiguous (n, 2) float32 tensor on the rays' device")
        n = rays.shape[0]
        out = _check_out(out, (n, 8), rays.device)
        _check(load_library().lsnif_query_pairs(self.h, rays.data_ptr(), intervals.data_ptr(), n, mode,
                                                out.data_ptr(), _stream_ptr(stream)))
        return out

    def last_stats(self, stream=None) -> dict:
        s = QueryStats()
        _check(load_library().lsnif_last_query_stats(self.h, _stream_ptr(stream), C.byref(s)))
        return {k: int(getattr(s, k)) for k, _ in QueryStats._fields_}

    def profile_enable(self, enable: bool = True) -> None:
        _check(load_library().lsnif_profile_enable(self.h, int(enable)))

    def profile_read(self, reset: bool = True, stream=None) -> dict:
        """Summed kernel durations / launch counts on `stream` (all streams if
        stream == 'all')."""
        p = Profile()
        sp = None if stream == "all" else _stream_ptr(stream)
        _check(load_library().lsnif_profile_read(self.h, sp, int(reset), C.byref(p)))
        return {k: getattr(p, k) for k, _ in Profile._fields_}

    def debug_traverse(self, rays) -> dict:
        torch = _torch()
        rays = rays.contiguous()
        n, H, L, F = rays.shape[0], self.H, self.n_levels, self.F
        dev = rays.device
        out = dict(info=torch.empty(n, dtype=torch.int32, device=dev),
                   interval=torch.empty((n, 2), dtype=torch.float32, device=dev),
                   t=torch.empty((n, H), dtype=torch.float32, device=dev),
                   pts=torch.empty((n, H, 3), dtype=torch.float32, device=dev),
                   cells=torch.empty((n, H), dtype=torch.int32, device=dev),
                   hidx=torch.empty((n, H, L, 8), dtype=torch.int32, device=dev),
                   feat=torch.empty((n, H * L * F), dtype=torch.float32, device=dev))
        _check(load_library().lsnif_debug_traverse(
            self.h, rays.data_ptr(), n, *[out[k].data_ptr() for k in
                                          ("info", "interval", "t", "pts", "cells", "hidx", "feat")],
            _stream_ptr(None)))
        return out

    def infer_batch(self, inputs, intervals, stream=None, exact: bool = False):
        """infer_batch (renderer.cpp:183-226). inputs: CUDA (n, input_width)
        fp32 — row j is column j of the reference's MatX; intervals (n, 2).
        The tcgen05 MLP (lsnif_infer_batch), or with exact=True the fp32
        kernel in the reference's summation order (lsnif_infer_batch_f32)."""
        torch = _torch()
        for name, t in (("inputs", inputs), ("intervals", intervals)):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float32 CUDA tensor (no implicit copies: a "
                                 "temporary could be freed before the asynchronous launch reads it)")
        n = inputs.shape[0]
        rows = inputs.shape[1] if inputs.dim() == 2 else 0
        out = torch.empty((n, 8), dtype=torch.int32, device=inputs.device)
        fn = load_library().lsnif_infer_batch_f32 if exact else load_library().lsnif_infer_batch
        _check(fn(self.h, inputs.data_ptr(), rows, n, intervals.data_ptr(), intervals.shape[0],
                  out.data_ptr(), _stream_ptr(stream)))
        return out

    # ---- host API (numpy, the reference's by-value vectors) ----
    def query_host(self, rays: np.ndarray, mode: int = CLOSEST, out: np.ndarray | None = None):
        rays = np.ascontiguousarray(rays)
        if rays.dtype != RAY_DTYPE:
            rays = rays.astype(np.float32, copy=False).reshape(-1, 8)
        n = len(rays)
        if out is None:
            out = np.empty(n, HIT_DTYPE)
        _check(load_library().lsnif_query_host(self.h, rays.ctypes.data, n, mode, out.ctypes.data,
                                               None))
        return out

    def query_host_wire(self, rays, mode: int = CLOSEST, out=None):
        """lsnif_query_host_wire: host rays (RAY_DTYPE / (n, 8) float32 array or
        pinned CPU tensor) -> WIRE_DTYPE records (or the given (n, 4) int32
        CPU tensor / WIRE_DTYPE array)."""
        if hasattr(rays, "data_ptr"):
            n, src = rays.shape[0], rays.data_ptr()
        else:
            rays = np.ascontiguousarray(rays)
            if rays.dtype != RAY_DTYPE:
                rays = rays.astype(np.float32, copy=False).reshape(-1, 8)
            n, src = len(rays), rays.ctypes.data
        if out is None:
            out = np.empty(n, WIRE_DTYPE)
        dst = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        _check(load_library().lsnif_query_host_wire(self.h, src, n, mode, dst, None))
        return out

    def intersect(self, rays: np.ndarray) -> np.ndarray:
        """Closest-hit narrow phase for one object (intersect_scene semantics)."""
        return self.query_host(rays, CLOSEST)

    def occluded(self, rays: np.ndarray) -> np.ndarray:
        """occluded_batch semantics: 1 where a neural hit lies in [t_min, t_max]."""
        h = self.query_host(rays, ANY)
        return ((h["flags_material"] & ACCEPTED) != 0).astype(np.int8)


class Camera(C.Structure):
    _fields_ = [("position", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("vfov_deg", C.c_float)]


class Light(C.Structure):
    _fields_ = [("type", C.c_uint32), ("position", C.c_float * 3), ("radius", C.c_float),
                ("radiance", C.c_float * 3)]


class RenderConfig(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("spp", C.c_int32),
                ("max_bounces", C.c_int32), ("seed", C.c_uint64), ("neural_eps_scale", C.c_float),
                ("max_paths_in_flight", C.c_int32)]


def _camera(camera: dict) -> Camera:
    c = Camera()
    c.position[:], c.look_at[:], c.up[:] = camera["position"], camera["look_at"], camera["up"]
    c.vfov_deg = camera["vfov_deg"]
    return c


def _config(cfg: dict) -> RenderConfig:
    r = RenderConfig()
    r.width, r.height, r.spp, r.max_bounces = cfg["width"], cfg["height"], cfg["spp"], cfg["max_bounces"]
    r.seed = int(cfg.get("seed", 0))
    r.neural_eps_scale = cfg.get("neural_eps_scale", 1e-3)
    r.max_paths_in_flight = int(cfg.get("max_paths_in_flight", 0))
    return r


def render_debug_paths(camera: dict, cfg: dict, first: int, n: int, k: int, device="cuda"):
    """GPU sampling probe: primary rays (n, 8) and the next k uniforms (n, k)."""
    torch = _torch()
    rays = torch.empty((n, 8), dtype=torch.float32, device=device)
    u = torch.empty((n, max(k, 1)), dtype=torch.float32, device=device)
    _check(load_library().lsnif_render_debug_paths(C.byref(_camera(camera)), C.byref(_config(cfg)),
                                                   first, n, rays.data_ptr(), u.data_ptr(), k,
                                                   _stream_ptr(None)))
    return rays, u[:, :k]


class RenderStats(C.Structure):
    _fields_ = [("paths", C.c_int64), ("closest_rays", C.c_int64), ("shadow_slots", C.c_int64),
                ("shadow_rays", C.c_int64), ("waves", C.c_int32), ("max_depth_reached", C.c_int32)]


class Instance(C.Structure):
    _fields_ = [("model", C.c_void_p), ("world_to_object", C.c_float * 12)]


class GpuScene:
    """Multi-object LSNIF scene: instances (model, world_to_object 3x4) in
    object order — the LSNIF part of PreparedScene (renderer.hpp:67-131)."""

    def __init__(self, instances):
        self._models = [m for m, _ in instances]  # keep the models alive
        arr = (Instance * len(instances))()
        for k, (m, w2o) in enumerate(instances):
            arr[k].model = m.h
            arr[k].world_to_object[:] = [float(v) for v in np.asarray(w2o, np.float32).reshape(12)]
        h = C.c_void_p()
        _check(load_library().lsnif_scene_create(arr, len(instances), C.byref(h)))
        self.h = h

    def query(self, rays, mode: int = CLOSEST, out=None, stream=None):
        """World-space CUDA rays (n, 8) -> (n, 16) int32 tensor of
        lsnif_scene_hit records (view with scene_hits_to_numpy)."""
        rays = _check_rays(rays)
        n = rays.shape[0]
        out = _check_out(out, (n, 16), rays.device)
        _check(load_library().lsnif_scene_query(self.h, rays.data_ptr(), n, mode, out.data_ptr(),
                                                _stream_ptr(stream)))
        return out

    def query_host(self, rays: np.ndarray, mode: int = CLOSEST, out: np.ndarray | None = None):
        """World-space HOST rays -> SCENE_HIT_DTYPE records (lsnif_scene_query_host:
        chunked H2D / scene query / D2H). Pinned arrays get the full PCIe rate;
        `rays` may be a RAY_DTYPE array or an (n, 8) float32 array/CPU tensor."""
        if hasattr(rays, "data_ptr"):
            n, src = rays.shape[0], rays.data_ptr()
        else:
            rays = np.ascontiguousarray(rays)
            if rays.dtype != RAY_DTYPE:
                rays = rays.astype(np.float32, copy=False).reshape(-1, 8)
            n, src = len(rays), rays.ctypes.data
        if out is None:
            out = np.empty(n, SCENE_HIT_DTYPE)
        dst = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        _check(load_library().lsnif_scene_query_host(self.h, src, n, mode, dst, None))
        return out

    def render(self, camera: dict, lights, environment, cfg: dict, world_diag, stream=None,
               stats: dict | None = None):
        """render() (renderer.cpp:453-542), PrimaryMode::lsnif: (H, W, 3) float32
        CUDA tensor, the spp-averaged image. `stats` (a dict) receives the ray
        counts of the call."""
        torch = _torch()
        n = len(world_diag)  # checked against the instance count by the library
        diag = (C.c_float * max(n, 1))(*[float(v) for v in world_diag])
        la = (Light * max(len(lights), 1))()
        for i, L in enumerate(lights):
            la[i].type = 1 if L["type"] == "sphere" else 0
            la[i].position[:] = L["position"]
            la[i].radius = L.get("radius", 0.0)
            la[i].radiance[:] = L["radiance"]
        env = (C.c_float * 3)(*[float(v) for v in environment])
        img = torch.empty((cfg["height"], cfg["width"], 3), dtype=torch.float32,
                          device=f"cuda:{self._models[0].device}")
        rs = RenderStats()
        _check(load_library().lsnif_render(self.h, diag, n, C.byref(_camera(camera)), la, len(lights),
                                           env, C.byref(_config(cfg)), img.data_ptr(), C.byref(rs),
                                           _stream_ptr(stream)))
        if stats is not None:
            stats.update({k: int(getattr(rs, k)) for k, _ in RenderStats._fields_})
        return img

    def close(self):
        if getattr(self, "h", None):
            load_library().lsnif_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scene_hits_to_numpy(hits) -> np.ndarray:
    a = hits.detach().cpu().numpy() if hasattr(hits, "detach") else np.asarray(hits)
    return np.ascontiguousarray(a).view(SCENE_HIT_DTYPE).reshape(-1)


def load_model(path: str, device: int = 0) -> GpuModel:
    return GpuModel(path, device)


def infer_batch(model: GpuModel, inputs, intervals):
    return model.infer_batch(inputs, intervals)


def hits_to_numpy(hits) -> np.ndarray:
    """(n, 8) int32 CUDA/CPU tensor of lsnif_hit -> numpy HIT_DTYPE records."""
    a = hits.detach().cpu().numpy() if hasattr(hits, "detach") else np.asarray(hits)
    return np.ascontiguousarray(a).view(HIT_DTYPE).reshape(-1)


def wire_to_hits(wire) -> np.ndarray:
    """Packed wire records ((n, 4) int32 tensor / WIRE_DTYPE array) -> HIT_DTYPE
    records, expanded by the library's host decode (lsnif_hits_from_wire)."""
    a = wire.detach().cpu().numpy() if hasattr(wire, "detach") else np.asarray(wire)
    a = np.ascontiguousarray(a).view(WIRE_DTYPE).reshape(-1)
    out = np.empty(len(a), HIT_DTYPE)
    _check(load_library().lsnif_hits_from_wire(a.ctypes.data, len(a), out.ctypes.data))
    return out


def rays_to_tensor(rays: np.ndarray, device="cuda"):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(rays).view(np.float32).reshape(-1, 8).copy()).to(device)


# ------------------------------------------------------------ GPU training (F4)

TARGET_DTYPE = np.dtype([("occluded", "<i4"), ("local_t", "<f4"), ("normal", "<f4", 3),
                         ("albedo", "<f4", 3), ("material", "<i4")])


class MeshDesc(C.Structure):
    _fields_ = [("vertices", C.c_void_p), ("n_vertices", C.c_int32), ("normals", C.c_void_p),
                ("n_normals", C.c_int32), ("faces", C.c_void_p), ("face_normals", C.c_void_p),
                ("face_material", C.c_void_p), ("n_faces", C.c_int32)]


class TrainConfig(C.Structure):
    _fields_ = [("batch", C.c_int32), ("lr", C.c_float), ("external_mix", C.c_float),
                ("seed", C.c_uint64)]


class TrainLoss(C.Structure):
    _fields_ = [("total", C.c_float), ("occlusion_bce", C.c_float), ("local_t_mae", C.c_float),
                ("normal_cosine", C.c_float), ("albedo_rel_l2", C.c_float), ("material_ce", C.c_float),
                ("step", C.c_int64)]


class _Loaded:  # wraps an exported lsnif_model handle as a GpuModel
    pass


class Trainer:
    """lsnif::train (training.cpp:95-230) on the GPU: mesh (verts (nv,3),
    faces (nf,3), optional normals / face_normals, face_material) + a
    starting LSNF file."""

    def __init__(self, init_path: str, mesh: dict, batch: int = 1 << 14, lr: float = 0.01,
                 external_mix: float = 0.5, seed: int = 0, device: int = 0):
        self._keep = {k: (np.ascontiguousarray(v, np.int32 if "face" in k else np.float32)
                          if v is not None else None) for k, v in mesh.items()}
        m = self._keep
        p = lambda a: a.ctypes.data if a is not None else None
        desc = MeshDesc(p(m["verts"]), len(m["verts"]), p(m.get("normals")),
                        0 if m.get("normals") is None else len(m["normals"]), p(m["faces"]),
                        p(m.get("face_normals")), p(m["face_material"]), len(m["faces"]))
        cfg = TrainConfig(batch, lr, external_mix, seed)
        h = C.c_void_p()
        _check(load_library().lsnif_trainer_create_from_file(init_path.encode(), C.byref(desc),
                                                             C.byref(cfg), device, C.byref(h)))
        self.h, self.device, self.batch = h, device, batch

    def step(self, steps: int = 1, stream=None) -> dict:
        loss = TrainLoss()
        _check(load_library().lsnif_trainer_step(self.h, steps, C.byref(loss), _stream_ptr(stream)))
        return {k: getattr(loss, k) for k, _ in TrainLoss._fields_}

    def sample(self, step: int, n: int):
        torch = _torch()
        rays = torch.empty((n, 8), dtype=torch.float32, device=f"cuda:{self.device}")
        tg = torch.empty((n, 9), dtype=torch.int32, device=f"cuda:{self.device}")
        _check(load_library().lsnif_trainer_sample(self.h, step, n, rays.data_ptr(), tg.data_ptr(),
                                                   _stream_ptr(None)))
        return rays, tg

    def batch_grad(self, rays, targets, n_mlp: int, n_tab: int):
        torch = _torch()
        g_mlp = torch.empty(n_mlp, dtype=torch.float32, device=rays.device)
        g_tab = torch.empty(n_tab, dtype=torch.float32, device=rays.device)
        loss = TrainLoss()
        _check(load_library().lsnif_trainer_batch_grad(self.h, rays.data_ptr(), targets.data_ptr(),
                                                       rays.shape[0], C.byref(loss), g_mlp.data_ptr(),
                                                       g_tab.data_ptr(), _stream_ptr(None)))
        return {k: getattr(loss, k) for k, _ in TrainLoss._fields_}, g_mlp, g_tab

    def export(self) -> "GpuModel":
        h = C.c_void_p()
        _check(load_library().lsnif_trainer_export(self.h, C.byref(h)))
        gm = GpuModel.__new__(GpuModel)
        gm.h, gm.device = h, self.device
        info = ModelInfo()
        _check(load_library().lsnif_model_get_info(gm.h, C.byref(info)))
        gm.info = info
        gm.H, gm.n_levels, gm.F = info.hit_cap, info.n_levels, info.f_dim
        gm.input_width = gm.H * gm.n_levels * gm.F
        gm.aabb = np.array(list(info.aabb), np.float32)
        return gm

    def close(self):
        if getattr(self, "h", None):
            load_library().lsnif_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
