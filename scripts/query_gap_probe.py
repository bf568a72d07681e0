"""Whole-query device time (CUDA events around lsnif_query) with and without
the library's per-kernel profiling events, vs the kernels' own durations."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
prim = W.camera_rays(1920, 1080)
hits = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(prim, "cuda")))
sets = {"c2": (lsnif.rays_to_tensor(prim, "cuda"), lsnif.CLOSEST),
        "c2shadow": (lsnif.rays_to_tensor(W.shadow_rays(prim, hits, gm.aabb)[0], "cuda"), lsnif.ANY)}
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for name, (d, mode) in sets.items():
    out = gm.query(d, mode)
    res = {"set": name}
    for prof in (False, True):
        gm.profile_enable(prof)
        gm.profile_read(reset=True)
        tot = 0.0
        for _ in range(20):
            flush.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gm.query(d, mode, out=out)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        p = gm.profile_read(reset=True)
        res["query_us_prof" if prof else "query_us"] = tot / 20 * 1e3
        if prof:
            res["kernels_us"] = (p["trace_ms"] + p["mlp_ms"]) / 20 * 1e3
    gm.profile_enable(False)
    print(json.dumps(res))
