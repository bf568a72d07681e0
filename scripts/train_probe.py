"""F4 probe: GPU training of the torus / sphere fixtures from their seed
init state — loss curve, ms per step (device events), held-out occlusion
accuracy of the exported binary16 model, and the oracle's batch-gradient
time per sample (one host thread) for scale."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2504_21627_b200 import lsnif  # noqa: E402

shape, name = (2, "torus_seed2") if (len(sys.argv) < 2 or sys.argv[1] == "torus") else (0, "sphere_seed1")
init = os.path.join(ROOT, "tests", "golden", name + ".lsnif")
verts, faces = O.shape_mesh(shape)
mesh = dict(verts=verts, faces=faces, face_material=np.zeros(len(faces), np.int32))
if shape == 0:
    mesh.update(normals=verts.copy(), face_normals=faces.copy())
batch = 1 << 14
tr = lsnif.Trainer(init, mesh, batch=batch, lr=0.01, seed=0)
rays, tg = tr.sample(step=10**7, n=1 << 16)
occ = tg.cpu().numpy().view(np.uint8).reshape(-1, 36).copy().view(lsnif.TARGET_DTYPE)["occluded"].reshape(-1)


def acc(model):
    h = lsnif.hits_to_numpy(model.query(rays))
    return float(np.mean(((h["flags_material"] & lsnif.OCCLUDED) != 0) == (occ != 0)))


out = {"fixture": name, "batch": batch, "faces": int(len(faces)), "acc_init": acc(lsnif.GpuModel(init)),
       "loss": []}
tr.step(1)
ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in range(10):
    ev[0].record()
    L = tr.step(50)
    ev[1].record()
    torch.cuda.synchronize()
    out["loss"].append((L["step"], round(L["total"], 5), round(L["occlusion_bce"], 5)))
    out["ms_per_step"] = ev[0].elapsed_time(ev[1]) / 50
out["acc_trained"] = acc(tr.export())
r = rays[:256].cpu().numpy().view(O.RAY_DTYPE).reshape(-1)
t = tg[:256].cpu().numpy().view(np.uint8).reshape(-1, 36).copy().view(O.TARGET_DTYPE).reshape(-1)
om = O.OracleModel.load(init)
t0 = time.perf_counter()
O.train_batch_grad(om, r, t)
out["oracle_us_per_sample_1thread"] = (time.perf_counter() - t0) / 256 * 1e6
out["gpu_us_per_sample"] = out["ms_per_step"] * 1e3 / batch
print(json.dumps(out))
