"""Runs one 2M-ray incoherent query on cuda:0 (after a warm-up) so the MLP
kernel's debug printf (LSNIF_MLP_DEBUG bit 2) reports an isolated launch."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2504_21627_b200 import lsnif, workloads as W
m = lsnif.GpuModel("tests/golden/teapot_seed0.lsnif")
r = lsnif.rays_to_tensor(W.incoherent_rays(1 << 21, m.aabb, seed=3))
m.query(r); torch.cuda.synchronize()
print("---- probe launch ----", flush=True)
m.profile_enable(True)
m.query(r); torch.cuda.synchronize()
print(m.profile_read(), flush=True)
