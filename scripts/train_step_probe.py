import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import oracle as O
from paper_2504_21627_b200 import lsnif
verts, faces = O.shape_mesh(2)
mesh = dict(verts=verts, faces=faces, face_material=np.zeros(len(faces), np.int32))
tr = lsnif.Trainer("/root/repo/tests/golden/torus_seed2.lsnif", mesh, batch=16384)
tr.step(3)
