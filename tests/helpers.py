"""Shared ray sets for the parity tests."""
import numpy as np

from paper_2504_21627_b200 import workloads as W


def edge_rays(box):
    """Hand-built edge cases: inside origins, axis-aligned and grid-plane
    origins, zero direction components, t_max gating, misses."""
    mn, mx = box[:3], box[3:]
    c = (mn + mx) / 2
    rs = []
    def add(o, d, t0=0.0, t1=np.inf):
        rs.append((np.array(o, np.float32), np.array(d, np.float32), t0, t1))
    add(c, (1, 0, 0)); add(c, (0, 1, 0)); add(c, (0, 0, -1))
    add(mn - 1, (1, 1, 1) / np.sqrt(3)); add(mx + 1, -np.ones(3) / np.sqrt(3))
    add((mn[0] - 1, c[1], c[2]), (1, 0, 0))           # axis aligned through the centre
    add((mn[0] - 1, mn[1], mn[2]), (1, 0, 0))         # along a box edge
    add((mn[0] - 1, c[1], c[2]), (-1, 0, 0))          # pointing away
    add((mn[0] - 1, c[1], c[2]), (1, 0, 0), 0.0, 0.5)  # t_max before the box: no pair
    add((mn[0] - 1, c[1], c[2]), (1, 0, 0), 2.0)       # t_min inside the box
    add(mn, (0.3, 0.4, 0.5)); add(mx, (-0.3, -0.4, -0.5))
    ext = mx - mn
    for k in range(32):                                # origins exactly on grid planes
        p = mn + ext * np.float32(k / 32)
        add(p, (0.6, 0.64, 0.48))
        add((p[0], c[1], c[2]), (0.0, 0.6, 0.8))
    rng = np.random.default_rng(7)
    for _ in range(200):                               # zero direction components
        d = rng.standard_normal(3).astype(np.float32)
        d[rng.integers(0, 3)] = 0.0
        add(rng.uniform(mn - 0.5, mx + 0.5).astype(np.float32), d / np.linalg.norm(d))
    out = np.zeros(len(rs), W.RAY_DTYPE)
    for i, (o, d, t0, t1) in enumerate(rs):
        out[i] = (o, d, t0, t1)
    return out


