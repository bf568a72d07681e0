"""Writes tests/golden/ref_teapot_vectors.npz from the REFERENCE ITSELF
(oracle/_ref: /root/reference/proj/src compiled against the Eigen-subset
shim, IEEE parity build). Run in the build container, where /root/reference
exists:  python tests/golden/make_ref_vectors.py

Contents (teapot_seed0.lsnif): 2,048 rays = 1,024 camera rays (C1 framing,
every 64th pixel) + 768 C5 incoherent rays + 256 edge-case rays;
  rays          (n, 8) float32 lsnif::Ray records
  hits_closest  (n, 8) uint32 narrow-phase records, closest-hit accept
  hits_any      (n, 8) uint32 the same with the any-hit accept
  info          (n,)   int32 count | first_is_origin << 8 | pair << 9
  interval_bits, t_bits, pts_bits, feat_bits, cells, hidx  (uint32 views)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import edge_rays  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2504_21627_b200 import workloads as W  # noqa: E402


def main():
    m = ref.RefModel(os.path.join(HERE, "teapot_seed0.lsnif"))
    cam = W.camera_rays(256, 256)[::64]
    inc = W.incoherent_rays_at(np.arange(0, 3840 * 2160 * 16, 172801, dtype=np.uint64)[:768], m.aabb, seed=5)
    edges = edge_rays(m.aabb)[:256]
    rays = np.concatenate([cam, inc, edges])
    tr = m.trace(rays)
    out = dict(rays=rays.view(np.float32).reshape(-1, 8),
               hits_closest=m.narrow_phase(rays, 0, 1).view(np.uint32).reshape(-1, 8),
               hits_any=m.narrow_phase(rays, 1, 1).view(np.uint32).reshape(-1, 8),
               info=tr["info"], cells=tr["cells"], hidx=tr["hidx"],
               interval_bits=tr["interval"].view(np.uint32), t_bits=tr["t"].view(np.uint32),
               pts_bits=tr["pts"].view(np.uint32), feat_bits=tr["feat"].view(np.uint32))
    path = os.path.join(HERE, "ref_teapot_vectors.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(rays), "rays")


if __name__ == "__main__":
    main()
