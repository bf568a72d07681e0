"""Reads the LSNIF_MLP_TIMELINE probe (CTA 0 clock64 stamps, 64 slots per
tile) after one query. Run with LSNIF_LIB pointing at a -DLSNIF_MLP_TIMELINE build.
Slots: 0/1/2 L1/L2/L3 issued, 3/4 h1/h2 ready seen by the MMA thread, 5 X +
accumulator ready seen, 8+e/16+e L1/L2 done seen by epilogue warp e, 24+e/32+e
h1/h2 published by warp e, 40+e L3 done seen, 48+e tile finished."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
which = sys.argv[1] if len(sys.argv) > 1 else "c3"
rays = W.incoherent_rays(1 << 21, gm.aabb, seed=3) if which == "c3" else W.camera_rays(1920, 1080)
mode = lsnif.CLOSEST
if which == "shadow":
    hits = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(rays, "cuda")))
    rays, mode = W.shadow_rays(rays, hits, gm.aabb)[0], lsnif.ANY
d = lsnif.rays_to_tensor(rays, "cuda")
gm.query(d, mode)
gm.query(d, mode)
torch.cuda.synchronize()
lib = lsnif.load_library()
buf = np.zeros(1 << 16, np.uint64)
assert lib.lsnif_probe_mlp_timeline(C.c_void_p(buf.ctypes.data), len(buf)) == 0
T = buf.reshape(-1, 64).astype(np.int64)
E = T[1023, :4].copy()  # CTA 0: entry, dependency resolved, weights in SMEM, all tiles done
T[1023] = 0
n = int(np.max(np.nonzero(T[:, 0])[0])) + 1
print("CTA 0: entry->griddep wait %d, wait->weights %d, weights->first L1 issue %d, first L1 -> all done %d "
      "(%d tiles), total %d cycles" % (E[1] - E[0], E[2] - E[1], T[0, 0] - E[2], E[3] - T[0, 0], n, E[3] - E[0]))
T = T[:n]
sl = T[4:n - 4]
def med(x):
    return int(np.median(x))
print("tiles", n, "cycles/tile:", med(np.diff(T[2:n - 2:2, 0])) // 2)
print("L1 issue -> all warps saw L1 (max):", med(sl[:, 8:16].max(1) - sl[:, 0]))
print("E1 per warp (seen->published) median over warps:", [med(sl[:, 24 + e] - sl[:, 8 + e]) for e in range(8)])
print("last h1 published -> MMA saw h1:", med(sl[:, 3] - sl[:, 24:32].max(1)), " -> L2 issued:", med(sl[:, 1] - sl[:, 3]))
print("E2 per warp:", [med(sl[:, 32 + e] - sl[:, 16 + e]) for e in range(8)])
print("last h2 published -> MMA saw h2:", med(sl[:, 4] - sl[:, 32:40].max(1)), " -> L3 issued:", med(sl[:, 2] - sl[:, 4]))
print("L3 issued -> L3 seen (max warps):", med(sl[:, 40:48].max(1) - sl[:, 2]))
print("L3 seen -> tile finished per warp:", [med(sl[:, 48 + e] - sl[:, 40 + e]) for e in range(8)])
print("tile finished (warp e) -> next L1 of the group seen:",
      [med(T[6:n - 4, 8 + e] - T[4:n - 6, 48 + e]) for e in range(8)])
print("acc/X ready seen -> L1 issued:", med(sl[:, 0] - sl[:, 5]))
