"""A/B timing of the query kernels: device time per query for C2 primaries and
C3 rays, per library build (LSNIF_LIB) and drain threshold (LSNIF_TRACE_DRAIN).
Usage: LSNIF_LIB=lib.so python scripts/trace_tune.py drain1[,drain2]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
libs = [os.environ.get("LSNIF_LIB", "default")]
drains = sys.argv[1].split(",") if len(sys.argv) > 1 else ["16"]
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

path = os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
res = []
for lib in libs:
    gm = lsnif.GpuModel(path, 0)
    prim = W.camera_rays(1920, 1080)
    hits = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(prim, "cuda")))
    sets = {"c1": lsnif.rays_to_tensor(W.camera_rays(256, 256), "cuda"),
            "c2": lsnif.rays_to_tensor(prim, "cuda"),
            "c2shadow": lsnif.rays_to_tensor(W.shadow_rays(prim, hits, gm.aabb)[0], "cuda"),
            "c3": lsnif.rays_to_tensor(W.incoherent_rays(1 << 22, gm.aabb, seed=3), "cuda")}
    for dr in drains:
        os.environ["LSNIF_TRACE_DRAIN"] = dr
        for name, d in sets.items():
            mode = lsnif.ANY if name == "c2shadow" else lsnif.CLOSEST
            out = gm.query(d, mode)
            st = gm.last_stats()
            gm.profile_enable(True)
            for _ in range(3):
                gm.query(d, mode, out=out)
            gm.profile_read(reset=True)
            reps = 10
            tot = 0.0
            for _ in range(reps):
                flush.add_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gm.query(d, mode, out=out)
                e1.record()
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            p = gm.profile_read(reset=True)
            gm.profile_enable(False)
            r = dict(lib=os.path.basename(lib), drain=int(dr), set=name, rays=d.shape[0],
                     trace_ms=p["trace_ms"] / reps, mlp_ms=p["mlp_ms"] / reps,
                     bin_ms=p.get("bin_ms", 0.0) / reps, sort=os.environ.get("LSNIF_RAY_SORT", ""))
            r["grays_s_trace"] = d.shape[0] / r["trace_ms"] / 1e6
            r["query_ms"] = tot / reps
            r["carve"] = os.environ.get("LSNIF_TRACE_CARVEOUT", "")
            r["blocks"] = os.environ.get("LSNIF_TRACE_BLOCKS", "")
            r["stats"] = st
            res.append(r)
            print(json.dumps(r), flush=True)
    gm.close()
