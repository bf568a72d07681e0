"""Generates tests/golden/ fixtures with the CPU oracle (run in the build
container, where /root/reference exists):

  teapot_seed0.lsnif  the reference train() setup state (T = 0) for
                      proj/assets/teapot.obj: LocalFrame::for_mesh, V=32
                      surface voxelization, random-init hash grid (M=2^17,
                      levels 64/128, F=3) and MLP (108-128-128-10) from seed 0,
                      saved in the LSNF v1 format (model_io.cpp:71-114).
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
