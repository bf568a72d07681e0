"""Synthetic ray workloads for the LSNIF query path.

All generators are index-addressable and deterministic, so every GPU rank can
regenerate exactly its own shard, and the GPU path and the CPU oracle consume
the same float32 ray file. Rays are the reference's `Ray` record
(geometry.hpp:11-18), 32 B AoS: origin f32x3, direction f32x3, t_min, t_max.

* camera rays: the reference pinhole camera (renderer.cpp:335-360) at pixel
  centres (u = v = 0.5 instead of a random jitter);
* incoherent rays: origins uniform in the model's frame box, directions
  uniform on S^2 (sampling.hpp:26-31), drawn from a splitmix64 counter RNG
  keyed by (seed, ray index) (types.hpp:25-39 mixing).
"""
from __future__ import annotations

import math

import numpy as np

RAY_DTYPE = np.dtype([("o", "<f4", 3), ("d", "<f4", 3), ("t_min", "<f4"), ("t_max", "<f4")])

# C1/C2 framing of the teapot fixture.
CAMERA = dict(position=(0.2505, 1.6, 4.5), look_at=(0.2505, 0.87, 0.0), up=(0.0, 1.0, 0.0),
              vfov_deg=40.0)
LIGHT = (3.0, 4.0, 3.0)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix_bits(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer (types.hpp:25-31), vectorised over uint64."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def counter_uniforms(seed: int, index: np.ndarray, k: int) -> np.ndarray:
    """k float32 uniforms in [0, 1) per index: 24-bit mantissas of
    mix(mix(mix(seed + c) ^ index) ^ j)."""
    with np.errstate(over="ignore"):
        base = _mix_bits(np.uint64(seed) + np.uint64(0x632BE59BD9B4E019))
        h = _mix_bits(base ^ index.astype(np.uint64))
        out = np.empty((len(index), k), np.float32)
        for j in range(k):
            v = _mix_bits(h ^ np.uint64(j + 1))
            out[:, j] = (v >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / (1 << 24))
    return out


def rank_jitter(rank: int) -> tuple[float, float]:
    """Sub-pixel sample position of a rank's frame: pixel centre for rank 0,
    a low-discrepancy offset otherwise (each GPU answers a different frame)."""
    if rank == 0:
        return (0.5, 0.5)
    return ((rank * 0.6180339887) % 1.0, (rank * 0.7548776662) % 1.0)


def camera_rays(width: int, height: int, rows: tuple[int, int] | None = None,
                camera: dict = CAMERA, jitter: tuple[float, float] = (0.5, 0.5)) -> np.ndarray:
    """Pinhole rays in row-major pixel order (renderer.cpp:346-360) with the
    sub-pixel sample at `jitter` (pixel centre by default). `rows` = (y0, y1)
    selects a row band (for tile sharding)."""
    f32 = np.float32
    pos = np.array(camera["position"], f32)
    fwd = np.array(camera["look_at"], f32) - pos
    fwd = fwd / np.sqrt(np.sum(fwd * fwd, dtype=f32))
    up = np.array(camera["up"], f32)
    right = np.cross(fwd, up).astype(f32)
    right = right / np.sqrt(np.sum(right * right, dtype=f32))
    upv = np.cross(right, fwd).astype(f32)
    half_h = f32(math.tan(0.5 * camera["vfov_deg"] * math.pi / 180.0))
    half_w = f32(half_h * f32(width) / f32(height))
    y0, y1 = rows if rows is not None else (0, height)
    py, px = np.meshgrid(np.arange(y0, y1, dtype=f32), np.arange(width, dtype=f32), indexing="ij")
    sx = (f32(2) * (px + f32(jitter[0])) / f32(width) - f32(1)).reshape(-1, 1)
    sy = (f32(1) - f32(2) * (py + f32(jitter[1])) / f32(height)).reshape(-1, 1)
    d = fwd + (sx * half_w) * right + (sy * half_h) * upv
    d = d / np.sqrt(np.sum(d * d, axis=1, keepdims=True, dtype=f32))
    rays = np.zeros(len(d), RAY_DTYPE)
    rays["o"] = pos
    rays["d"] = d.astype(f32)
    rays["t_min"] = 0.0
    rays["t_max"] = np.inf
    return rays


def incoherent_rays(n: int, box: np.ndarray, seed: int = 3, start: int = 0) -> np.ndarray:
    """C3/C5 rays [start, start+n): origin uniform in `box` (min xyz, max xyz),
    direction uniform on the sphere (sampling.hpp:26-31)."""
    f32 = np.float32
    box = np.asarray(box, f32)
    idx = np.arange(start, start + n, dtype=np.uint64)
    u = counter_uniforms(seed, idx, 5)
    mn, mx = box[:3], box[3:]
    o = mn + u[:, :3] * (mx - mn)
    z = f32(1) - f32(2) * u[:, 3]
    r = np.sqrt(np.maximum(f32(0), f32(1) - z * z))
    phi = f32(2 * math.pi) * u[:, 4]
    rays = np.zeros(n, RAY_DTYPE)
    rays["o"] = o
    rays["d"] = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1).astype(f32)
    rays["t_min"] = 0.0
    rays["t_max"] = np.inf
    return rays


def incoherent_rays_at(idx: np.ndarray, box: np.ndarray, seed: int = 3) -> np.ndarray:
    """incoherent_rays for arbitrary ray indices (a strided CPU-baseline
    sample draws exactly the rays the GPU answers at those indices)."""
    f32 = np.float32
    box = np.asarray(box, f32)
    u = counter_uniforms(seed, np.asarray(idx, np.uint64), 5)
    mn, mx = box[:3], box[3:]
    o = mn + u[:, :3] * (mx - mn)
    z = f32(1) - f32(2) * u[:, 3]
    r = np.sqrt(np.maximum(f32(0), f32(1) - z * z))
    phi = f32(2 * math.pi) * u[:, 4]
    rays = np.zeros(len(u), RAY_DTYPE)
    rays["o"] = o
    rays["d"] = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1).astype(f32)
    rays["t_min"] = 0.0
    rays["t_max"] = np.inf
    return rays


def incoherent_rays_into(out: np.ndarray, box: np.ndarray, seed: int, start: int,
                         threads: int | None = None, chunk: int = 1 << 20) -> np.ndarray:
    """Fills `out` (RAY_DTYPE, or any (n, 8) float32 view of the same bytes)
    with incoherent_rays(len(out), box, seed, start), chunked over a thread
    pool (numpy releases the GIL: C5's 132.7M rays in seconds, not a minute).
    Bit-identical to incoherent_rays: every ray depends on its index only."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    view = np.asarray(out).view(np.float32).reshape(-1, 8)
    n = view.shape[0]

    def fill(s):
        e = min(n, s + chunk)
        view[s:e] = incoherent_rays(e - s, box, seed=seed, start=start + s).view(np.float32).reshape(-1, 8)

    workers = threads or max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(workers) as ex:
        list(ex.map(fill, range(0, n, chunk)))
    return out


def shadow_rays(primary: np.ndarray, hits: np.ndarray, box: np.ndarray,
                light=LIGHT, eps_scale: float = 1e-3) -> tuple[np.ndarray, np.ndarray]:
    """One NEE shadow ray per accepted neural hit (renderer.cpp:384-427 at
    identity transform, diffuse material, one point light): spawn at
    hit + eps*n with eps = 1e-3 * frame diagonal, normal from the head (or -d
    when zero) flipped to face the ray, kept iff n.wi > 0, t_max = 0.9999*dist.
    Returns (rays, owner index)."""
    f32 = np.float32
    acc = (hits["flags_material"] & 4) != 0
    idx = np.nonzero(acc)[0]
    o = primary["o"][idx]
    d = primary["d"][idx]
    t = hits["t_world"][idx].reshape(-1, 1)
    pos = o + t * d
    n = hits["normal"][idx].astype(f32)
    zero = np.sum(n * n, axis=1) == 0
    n[zero] = -d[zero]
    flip = np.sum(n * d, axis=1) > 0
    n[flip] = -n[flip]
    box = np.asarray(box, f32)
    diag = f32(np.sqrt(np.sum((box[3:] - box[:3]) ** 2)))
    spawn = pos + f32(eps_scale) * diag * n
    to_l = np.asarray(light, f32) - spawn
    dist = np.sqrt(np.sum(to_l * to_l, axis=1))
    wi = to_l / dist.reshape(-1, 1)
    keep = (np.sum(n * wi, axis=1) > 0) & (dist > 0)
    rays = np.zeros(int(keep.sum()), RAY_DTYPE)
    rays["o"] = spawn[keep]
    rays["d"] = wi[keep]
    rays["t_min"] = 0.0
    rays["t_max"] = dist[keep] * f32(1 - 1e-4)
    return rays, idx[keep]


# ---------------------------------------------------------------- C4 scene

C4_MODELS = ["teapot_seed0", "sphere_seed1", "torus_seed2", "box_seed3"]
C4_INSTANCES = [0, 1, 2, 3, 2, 0, 1, 0]   # model per instance: teapot x3, sphere x2, torus x2, box
C4_CAMERA = dict(position=(0.0, 7.0, 16.0), look_at=(0.0, 0.5, 0.0), up=(0.0, 1.0, 0.0),
                 vfov_deg=45.0)


def c4_world_to_object() -> np.ndarray:
    """(8, 3, 4) float32 world_to_object of the C4 instances: a 4x2 grid with
    4-unit spacing, yaw 0 / 45 degrees alternating."""
    out = np.zeros((8, 3, 4), np.float32)
    for i in range(8):
        pos = np.array([(i % 4 - 1.5) * 4.0, 0.0, (i // 4 - 0.5) * 4.0])
        yaw = math.radians(45.0 if i % 2 else 0.0)
        c, s = math.cos(yaw), math.sin(yaw)
        R = np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])   # object -> world rotation
        Rt = R.T                                            # world -> object
        out[i, :, :3] = Rt
        out[i, :, 3] = -Rt @ pos
    return out


def c4_bounds() -> np.ndarray:
    return np.array([-8.5, -1.5, -4.5, 8.5, 2.5, 4.5], np.float32)


# ------------------------------------------------------- render scene (F3)

RENDER_MODELS = ["teapot_seed0", "sphere_seed1", "box_seed3", "torus_seed2"]
RENDER_CAMERA = dict(position=(0.0, 2.2, 7.0), look_at=(0.0, 0.5, 0.0), up=(0.0, 1.0, 0.0),
                     vfov_deg=40.0)
RENDER_LIGHTS = [dict(type="point", position=(3.0, 4.0, 3.0), radiance=(20.0, 20.0, 20.0)),
                 dict(type="sphere", position=(-2.5, 3.5, 2.0), radius=0.5,
                      radiance=(8.0, 8.0, 8.0))]
RENDER_ENV = (0.05, 0.05, 0.08)
RENDER_PLACEMENT = [(0.0, 0.0, 0.0), (2.6, 0.6, 0.3), (-2.6, 0.6, 0.2), (0.0, 0.35, -2.4)]


def render_world_to_object() -> np.ndarray:
    """(4, 3, 4) world_to_object of the render scene: translations (pure
    translation keeps the frame box axis-aligned in the world)."""
    out = np.zeros((len(RENDER_PLACEMENT), 3, 4), np.float32)
    for i, p in enumerate(RENDER_PLACEMENT):
        out[i, :, :3] = np.eye(3)
        out[i, :, 3] = -np.asarray(p, np.float32)
    return out


def world_diag_from_frames(aabbs) -> list[float]:
    """PreparedObject::world_diag stand-in: the diagonal of each instance's
    frame box (the mesh bounds are not part of the model file; translation
    only, so world and object diagonals agree)."""
    out = []
    for a in aabbs:
        a = np.asarray(a, np.float32)
        e = a[3:] - a[:3]
        out.append(float(np.float32(np.sqrt(np.float32((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2])))))
    return out


def glossy_copy(src: str, dst: str, material: int, roughness: float) -> str:
    """Copies an LSNF v1 file, switching material slot `material` to glossy
    (MaterialKind 1) with `roughness` — to exercise shade_hit's Phong branch."""
    import struct
    b = bytearray(open(src, "rb").read())
    for n in range(1, 65):  # material block: u32 count, n x {3 f32 albedo, u32 kind, f32 rough}
        off = len(b) - 24 - 20 * n - 4
        if off > 0 and struct.unpack_from("<I", b, off)[0] == n:
            break
    else:
        raise ValueError("no material table found")
    assert 0 <= material < n
    struct.pack_into("<If", b, off + 4 + 20 * material + 12, 1, roughness)
    open(dst, "wb").write(bytes(b))
    return dst
