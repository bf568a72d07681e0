"""One C4 scene query (8 instances, 1080p camera rays) after a warm-up, for ncu launch lists."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gold = os.path.join(ROOT, "tests", "golden")
models = [lsnif.GpuModel(os.path.join(gold, n + ".lsnif")) for n in W.C4_MODELS]
w2o = W.c4_world_to_object()
scene = lsnif.GpuScene([(models[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
d = lsnif.rays_to_tensor(W.camera_rays(1920, 1080, camera=W.C4_CAMERA), "cuda")
out = scene.query(d, 0)
torch.cuda.synchronize()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    scene.query(d, 0, out=out)
torch.cuda.synchronize()
