"""Host-API (lsnif_query_host) throughput on the C2 primaries vs the staging
chunk size (LSNIF_HOST_CHUNK, read when a model's staging is created)."""
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
rays = W.camera_rays(1920, 1080)
n = len(rays)
pin_r = torch.from_numpy(rays.view(np.float32).reshape(-1, 8).copy()).pin_memory()
pin_h = torch.empty((n, 8), dtype=torch.int32).pin_memory()
lib = lsnif.load_library()
for chunk in (sys.argv[1] if len(sys.argv) > 1 else "65536,131072,262144,524288").split(","):
    os.environ["LSNIF_HOST_CHUNK"] = chunk
    gm = lsnif.GpuModel(path, 0)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lsnif._check(lib.lsnif_query_host(gm.h, pin_r.data_ptr(), n, lsnif.CLOSEST, pin_h.data_ptr(), st))
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        lsnif._check(lib.lsnif_query_host(gm.h, pin_r.data_ptr(), n, lsnif.CLOSEST, pin_h.data_ptr(), st))
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"chunk": int(chunk), "ms": dt * 1e3, "rays_per_s": n / dt,
                      "pcie_GBps_each_way": n * 32 / dt / 1e9}), flush=True)
    gm.close()
