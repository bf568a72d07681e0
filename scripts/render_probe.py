"""One render of the F3 bench scene (for ncu launch lists / timing probes)."""
import os
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

w, h = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "640x360").split("x"))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
paths = bench.render_scene_paths(tempfile.mkdtemp())
models = [lsnif.GpuModel(p) for p in paths]
w2o = W.render_world_to_object()
scene = lsnif.GpuScene([(models[i], w2o[i]) for i in range(len(models))])
diag = W.world_diag_from_frames([m.aabb for m in models])
cfg = dict(bench.RENDER_CFG, width=w, height=h)
st = {}
scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag, stats=st)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag, stats=st)
torch.cuda.synchronize()
print(st, f"{(time.perf_counter() - t0) / reps * 1e3:.2f} ms per render")
