"""Host-API (lsnif_query_host) timing on the C2 rays: primary, shadow and the
bench's primary+shadow step, vs the staging chunk size (LSNIF_HOST_CHUNK)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

path = os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif")
prim = W.camera_rays(1920, 1080)
gm0 = lsnif.GpuModel(path, 0)
d = lsnif.rays_to_tensor(prim, "cuda")
hits = lsnif.hits_to_numpy(gm0.query(d))
shadow, _ = W.shadow_rays(prim, hits, gm0.aabb)
gm0.close()
lib = lsnif.load_library()


def pinned(rays):
    r = torch.from_numpy(rays.view(np.float32).reshape(-1, 8).copy()).pin_memory()
    return r, torch.empty((len(rays), 8), dtype=torch.int32).pin_memory()


pr, ph = pinned(prim)
sr, sh = pinned(shadow)
for chunk in (sys.argv[1] if len(sys.argv) > 1 else "131072").split(","):
    os.environ["LSNIF_HOST_CHUNK"] = chunk
    gm = lsnif.GpuModel(path, 0)

    def q(r, h, n, mode):
        lsnif._check(lib.lsnif_query_host(gm.h, r.data_ptr(), n, mode, h.data_ptr(), None))

    cases = {"primary": lambda: q(pr, ph, len(prim), lsnif.CLOSEST),
             "shadow": lambda: q(sr, sh, len(shadow), lsnif.ANY),
             "step": lambda: (q(pr, ph, len(prim), lsnif.CLOSEST), q(sr, sh, len(shadow), lsnif.ANY))}
    out = {"chunk": int(chunk)}
    for name, fn in cases.items():
        for _ in range(3):
            fn()
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        out[name + "_ms"] = (time.perf_counter() - t0) / reps * 1e3
    out["step_rays_per_s"] = (len(prim) + len(shadow)) / out["step_ms"] * 1e3
    print(json.dumps(out), flush=True)
    gm.close()
