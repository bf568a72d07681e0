"""Device time per training step (sampler + encode + forward/backward +
scatter + Adam) on the torus fixture at a given batch, CUDA events around
`steps` steps after 2 warm-up steps. Usage: python scripts/train_time.py [batch] [steps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2504_21627_b200 import lsnif  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
verts, faces = O.shape_mesh(2)
mesh = dict(verts=verts, faces=faces, face_material=np.zeros(len(faces), np.int32))
tr = lsnif.Trainer(os.path.join(ROOT, "tests", "golden", "torus_seed2.lsnif"), mesh, batch=batch)
tr.step(2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
loss = tr.step(steps)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(json.dumps({"lib": os.path.basename(lsnif.LIB_PATH), "batch": batch, "ms_per_step": ms,
                  "rays_per_s": batch / ms * 1e3, "loss": loss["total"]}))
