"""Device time of lsnif_infer_batch (tcgen05 MLP) vs lsnif_infer_batch_f32 on
encoded columns of incoherent teapot rays (oracle encode), CUDA events.
Usage: python scripts/infer_time.py [n_rays]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
path = os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif")
gm, om = lsnif.GpuModel(path, 0), O.OracleModel.load(path)
tr = om.trace(W.incoherent_rays(n, gm.aabb, seed=21))
keep = (tr["info"] >> 9) & 1 == 1
x = torch.from_numpy(tr["feat"][keep]).cuda()
iv = torch.from_numpy(tr["interval"][keep]).cuda()
res = {"columns": int(x.shape[0])}
for name, exact in (("tcgen05", False), ("fp32", True)):
    gm.infer_batch(x, iv, exact=exact)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        gm.infer_batch(x, iv, exact=exact)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = {"ms": ms, "columns_per_s": x.shape[0] / ms * 1e3,
                 "tflops": x.shape[0] * 62976 / ms / 1e9}
print(json.dumps(res))
