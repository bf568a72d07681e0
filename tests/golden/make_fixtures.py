"""Generates tests/golden/ fixtures with the CPU oracle (run in the build
container, where /root/reference exists):

  teapot_seed0.lsnif  the reference train() setup state (T = 0) for
                      proj/assets/teapot.obj: LocalFrame::for_mesh, V=32
                      surface voxelization, random-init hash grid (M=2^17,
                      levels 64/128, F=3) and MLP (108-128-128-10) from seed 0,
                      saved in the LSNF v1 format (model_io.cpp:71-114).
  sphere_seed1.lsnif, torus_seed2.lsnif, box_seed3.lsnif
                      the same setup state for the procedural fixtures of
                      shapes.cpp (make_uv_sphere(1,32,16), make_torus(1,.35,48,24),
                      make_box((1,.6,.8))) with seeds 1, 2, 3 — the C4 scene's
                      other objects.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle  # noqa: E402

REF_OBJ = "/root/reference/proj/assets/teapot.obj"

if __name__ == "__main__":
    out = os.path.join(HERE, "teapot_seed0.lsnif")
    oracle.build_obj_model(REF_OBJ, out, V=32, H=18, seed=0)
    print("wrote", out, os.path.getsize(out), "bytes")
    for shape, seed, name in [(0, 1, "sphere_seed1"), (2, 2, "torus_seed2"), (1, 3, "box_seed3")]:
        p = os.path.join(HERE, name + ".lsnif")
        oracle.build_shape_model(shape, seed, p)
        print("wrote", p, os.path.getsize(p), "bytes")
