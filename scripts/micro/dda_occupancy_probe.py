"""Walk-only kernel at 32 / 48 / 64 warps per SM on C3 rays, in input order and
sorted by estimated walk length (scripts/micro/dda_occupancy_probe.cuh; needs
the A/B build `bash scripts/build_variant.sh probe -DLSNIF_PROBE`)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("LSNIF_LIB", os.path.join(ROOT, "ab", "probe.so"))
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"), 0)
lib = lsnif.load_library()
lib.lsnif_probe_dda.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.POINTER(C.c_float)]
rays = W.incoherent_rays(1 << 22, gm.aabb, seed=3)
r = rays.view(np.float32).reshape(-1, 8)
mn, mx = gm.aabb[:3], gm.aabb[3:]
lo = (r[:, 0:3] - mn) / (mx - mn)
ld = r[:, 3:6] / (mx - mn)
with np.errstate(divide="ignore", invalid="ignore"):
    ta, tb = -lo / ld, (1 - lo) / ld
    t0 = np.maximum(r[:, 6], np.nanmax(np.minimum(ta, tb), axis=1))
    t1 = np.nanmin(np.maximum(ta, tb), axis=1)
    c0 = np.floor((lo + t0[:, None] * ld) * 32)
    c1 = np.floor((lo + t1[:, None] * ld) * 32)
    est = np.where(t0 < t1, np.abs(c1 - c0).sum(axis=1), -1)
order = np.argsort(-est, kind="stable")
sets = {"input order": rays, "walk-length order": rays[order]}
out = torch.empty(len(rays), dtype=torch.int32, device="cuda")
res = []
for name, rs in sets.items():
    d = lsnif.rays_to_tensor(rs, "cuda")
    for wps in (32, 48, 64):
        ms = C.c_float()
        best = 1e9
        for _ in range(5):
            rc = lib.lsnif_probe_dda(gm.h, d.data_ptr(), len(rs), out.data_ptr(), wps, C.byref(ms))
            assert rc == 0, rc
            best = min(best, ms.value)
        res.append({"rays": name, "warps_per_sm": wps, "walk_us": best * 1e3})
        print(json.dumps(res[-1]), flush=True)
