"""Minimal debug_traverse / query repro for compute-sanitizer runs."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402
gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
rays = lsnif.rays_to_tensor(W.camera_rays(int(sys.argv[1]) if len(sys.argv) > 1 else 64, 64), "cuda")
out = gm.debug_traverse(rays)
print({k: v.shape for k, v in out.items()})
big = lsnif.rays_to_tensor(W.incoherent_rays(640 * 1024, gm.aabb, seed=5), "cuda")
h = gm.query(big, lsnif.CLOSEST)
print("query ok", h.shape)
