"""A/B of the scene path between two library builds: dumps the C4 scene hits
(camera + incoherent, closest + any) and times the C4 query.
Usage: LSNIF_LIB=x.so python scripts/scene_ab.py out.npz"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gold = os.path.join(ROOT, "tests", "golden")
models = [lsnif.GpuModel(os.path.join(gold, n + ".lsnif")) for n in W.C4_MODELS]
w2o = W.c4_world_to_object()
scene = lsnif.GpuScene([(models[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
cam = lsnif.rays_to_tensor(W.camera_rays(1920, 1080, camera=W.C4_CAMERA), "cuda")
inc = lsnif.rays_to_tensor(W.incoherent_rays(1 << 20, W.c4_bounds(), seed=4), "cuda")
res = {}
for name, d in (("cam", cam), ("inc", inc)):
    for mode in (0, 1):
        res[f"{name}{mode}"] = scene.query(d, mode).cpu().numpy()
np.savez(sys.argv[1], **res)
out = scene.query(cam, 0)
for _ in range(5):
    scene.query(cam, 0, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    scene.query(cam, 0, out=out)
e1.record()
torch.cuda.synchronize()
print(os.path.basename(os.environ.get("LSNIF_LIB", "default")), "C4 query ms", e0.elapsed_time(e1) / 20)
