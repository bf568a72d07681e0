"""C2 shadow-ray query in isolation: per-kernel device times (library
profile events) of the ANY-mode query on the NEE shadow rays, and the
points/volume-point mix. Under ncu: launches are primary trace, primary MLP,
then shadow trace / MLP pairs."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
prim = W.camera_rays(1920, 1080)
hits = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(prim, "cuda")))
sh = W.shadow_rays(prim, hits, gm.aabb)[0]
if len(sys.argv) > 1 and sys.argv[1] == "shuffle":
    sh = sh[np.random.default_rng(0).permutation(len(sh))]
d = lsnif.rays_to_tensor(sh, "cuda")
out = gm.query(d, lsnif.ANY)
st = gm.last_stats()
gm.profile_enable(True)
reps = 20
for _ in range(reps):
    gm.query(d, lsnif.ANY, out=out)
torch.cuda.synchronize()
p = gm.profile_read(reset=True)
print(json.dumps({"rays": len(sh), "trace_us": 1e3 * p["trace_ms"] / reps, "mlp_us": 1e3 * p["mlp_ms"] / reps,
                  "stats": st}), flush=True)
