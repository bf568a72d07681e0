"""e2e timing of lsnif_scene_query_host on the C4 scene (pinned buffers),
against the device-only scene query and a copy-only round trip.
Usage: LSNIF_HOST_CHUNK=<rays> python scripts/scene_e2e_probe.py"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gold = os.path.join(ROOT, "tests", "golden")
models = [lsnif.GpuModel(os.path.join(gold, n + ".lsnif")) for n in W.C4_MODELS]
w2o = W.c4_world_to_object()
scene = lsnif.GpuScene([(models[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
rays = W.camera_rays(1920, 1080, camera=W.C4_CAMERA)
pin_r = torch.from_numpy(rays.view(np.float32).reshape(-1, 8).copy()).pin_memory()
pin_h = torch.empty((len(rays), 16), dtype=torch.int32).pin_memory()
d_r = pin_r.cuda()
d_h = torch.empty((len(rays), 16), dtype=torch.int32, device="cuda")


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


res = {"chunk": os.environ.get("LSNIF_HOST_CHUNK", "default"),
       "host_ms": t(lambda: scene.query_host(pin_r, lsnif.CLOSEST, out=pin_h)),
       "device_ms": t(lambda: scene.query(d_r, lsnif.CLOSEST, out=d_h)),
       "copy_ms": t(lambda: (d_r.copy_(pin_r, non_blocking=True), pin_h.copy_(d_h, non_blocking=True)))}
print(json.dumps(res), flush=True)
