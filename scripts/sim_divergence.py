"""DDA lane-efficiency model for incoherent rays (C3 distribution, teapot):
per-ray walk lengths from a numpy restatement of the dda.cpp:88-116 stepping,
then the fraction of useful lane-steps when 32-lane warps walk rays in
arrival order vs in rounds regrouped by (true / estimated) walk length within
runs of 64-256 rays. Motivates the sorted runs of trace_encode_kernel.
Usage: python scripts/sim_divergence.py"""
import sys, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle import oracle as O
from paper_2504_21627_b200 import workloads as W
om = O.OracleModel.load(__import__("os").path.join(sys.path[0], "tests", "golden", "teapot_seed0.lsnif"))
V=om.V; H=om.H
occ = np.unpackbits(om.occupancy(), bitorder="little").astype(bool)  # idx = x + V(y + V z)
n = 1<<17
rays = W.incoherent_rays(n, om.aabb, seed=3)
box = om.aabb.astype(np.float64)
o = (rays["o"] - box[:3]) / (box[3:] - box[:3]); d = rays["d"] / (box[3:] - box[:3])
# slab in unit cube
with np.errstate(divide="ignore", invalid="ignore"):
    inv = 1/d
    ta = (0 - o)*inv; tb = (1 - o)*inv
t0 = np.maximum(np.max(np.minimum(ta, tb), 1), 0); t1 = np.min(np.maximum(ta, tb), 1)
ok = t0 <= t1
start = o + t0[:,None]*d
c = np.clip(np.floor(start*V).astype(int), 0, V-1)
step = np.sign(d).astype(int)
with np.errstate(divide="ignore", invalid="ignore"):
    td = np.abs(1/(V*d))
    nxt = np.where(d>0, (c+1)/V, c/V)
    tn = np.where(d!=0, t0[:,None] + (nxt - start)/d, np.inf)
alive = ok.copy(); cnt = np.zeros(n, int); steps = np.zeros(n, int)
lin = lambda c: c[:,0] + V*(c[:,1] + V*c[:,2])
inside = lambda c: np.all((c>=0)&(c<V),1)
first = alive & occ[lin(np.clip(c,0,V-1))]
cnt += first
while alive.any():
    ax = np.argmin(tn, 1)  # ties: lowest axis (matches strict <)
    t = tn[np.arange(n), ax]
    stop = alive & ((t > t1) | (cnt >= H))
    alive &= ~stop
    r = np.arange(n)[alive]
    a = ax[alive]
    c[r, a] += step[r, a]; tn[r, a] += td[r, a]; steps[r] += 1
    ins = inside(c[r])
    alive[r[~ins]] = False
    rr = r[ins]
    hit = occ[lin(c[rr])]
    cnt[rr[hit]] += 1
print("mean steps", steps.mean(), "max", steps.max(), "mean pts", cnt.mean())
s = steps.reshape(-1, 32)
eff = s.mean() / s.max(1).mean()
print("batch-32 DDA efficiency", eff, "iters/warp", s.max(1).mean())
for S in (64, 128, 256):
    g = np.sort(steps.reshape(-1, S), 1).reshape(-1, S//32, 32)
    print(S, "sorted efficiency", g.mean() / g.max(2).mean(), "iters per 32", g.max(2).mean())
# points encode passes
p = cnt.reshape(-1,32).sum(1)
print("encode passes/warp", np.ceil(p/32).mean(), "pts/warp", p.mean())
end = o + t1[:,None]*d
ce = np.clip(np.floor(end*V).astype(int), -1, V)
est = np.abs(ce - np.clip(np.floor(start*V).astype(int), 0, V-1)).sum(1)
print("corr", np.corrcoef(est, steps)[0,1])
for S in (128, 256):
    idx = np.argsort(est.reshape(-1, S), 1, kind="stable")
    g = np.take_along_axis(steps.reshape(-1, S), idx, 1).reshape(-1, S//32, 32)
    print(S, "est-sorted efficiency", g.mean() / g.max(2).mean(), "iters per 32", g.max(2).mean())
    # points per round
    pc = np.take_along_axis(cnt.reshape(-1, S), idx, 1).reshape(-1, S//32, 32).sum(2)
    print("  encode passes per round", np.ceil(pc/32).mean(), "pts", pc.mean())
