"""Small end-to-end exercise of every kernel family for compute-sanitizer:
query (trace + MLP; in-kernel clip, given pair intervals, host staging; one
launch large enough for the 1024-thread / byte-mask trace configuration),
debug traverse, infer_batch, scene query (device and host), render, and two
training steps."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2504_21627_b200 import lsnif, workloads as W  # noqa: E402

gold = os.path.join(ROOT, "tests", "golden")
gm = lsnif.GpuModel(os.path.join(gold, "teapot_seed0.lsnif"))
rays = lsnif.rays_to_tensor(np.concatenate([W.camera_rays(64, 48), W.incoherent_rays(4096, gm.aabb, seed=3)]), "cuda")
gm.query(rays, lsnif.CLOSEST)
gm.query(rays, lsnif.ANY)
gm.debug_traverse(rays[:512])
big = lsnif.rays_to_tensor(W.incoherent_rays(640 * 1024, gm.aabb, seed=5), "cuda")  # >= 4 waves: 1024-thread blocks
gm.query(big, lsnif.CLOSEST)
ivs = torch.rand((rays.shape[0], 2), device="cuda").sort(dim=1).values * 4  # given pair intervals
gm.query_pairs(rays, ivs, lsnif.CLOSEST)
gm.query_host(rays.cpu().numpy().view(lsnif.RAY_DTYPE).reshape(-1), lsnif.ANY)
x = torch.zeros((64, gm.input_width), dtype=torch.float32, device="cuda")
iv = torch.zeros((64, 2), dtype=torch.float32, device="cuda")
gm.infer_batch(x, iv)                          # tcgen05 MLP (infer_pack_kernel + mlp_tc_kernel)
gm.infer_batch(x, iv, exact=True)              # fp32 kernel
gm.infer_batch(torch.full_like(x, 1e6), iv)    # out-of-range inputs: the device-side fp32 fallback
models = [lsnif.GpuModel(os.path.join(gold, n + ".lsnif")) for n in W.RENDER_MODELS]
w2o = W.render_world_to_object()
scene = lsnif.GpuScene([(models[i], w2o[i]) for i in range(len(models))])
scene.query(lsnif.rays_to_tensor(W.camera_rays(32, 24, camera=W.RENDER_CAMERA), "cuda"))
scene.query_host(W.camera_rays(40, 30, camera=W.RENDER_CAMERA), lsnif.ANY)
img = scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, dict(width=24, height=16, spp=2, max_bounces=2),
                   W.world_diag_from_frames([m.aabb for m in models]))
verts, faces = O.shape_mesh(0)
tr = lsnif.Trainer(os.path.join(gold, "sphere_seed1.lsnif"),
                   dict(verts=verts, faces=faces, face_material=np.zeros(len(faces), np.int32)), batch=512)
tr.step(2)
tr.export().query(rays[:256])
torch.cuda.synchronize()
print("sanitize probe ok", float(img.mean()))
