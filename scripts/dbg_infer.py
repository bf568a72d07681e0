import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import oracle as O
from paper_2504_21627_b200 import lsnif, workloads as W
m = O.OracleModel.load('tests/golden/teapot_seed0.lsnif')
g = lsnif.GpuModel('tests/golden/teapot_seed0.lsnif')
rays = W.incoherent_rays(8192, g.aabb, seed=11)
tr = m.trace(rays)
keep = (tr["info"] >> 9) & 1 == 1
x, iv = tr["feat"][keep], tr["interval"][keep]
ref = m.infer_batch(x, iv)
got = lsnif.hits_to_numpy(g.infer_batch(torch.from_numpy(x).cuda(), torch.from_numpy(iv).cuda()))
os.makedirs('gpurun_out', exist_ok=True)
np.savez('gpurun_out/infer_dbg.npz', x=x, iv=iv, ref=ref.view(np.uint32).reshape(-1,8), got=got.view(np.uint32).reshape(-1,8))
bad = np.nonzero(got['flags_material'] != ref['flags_material'])[0]
print('mismatch', len(bad), bad[:10], got['flags_material'][bad[:10]], ref['flags_material'][bad[:10]])
