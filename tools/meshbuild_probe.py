import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2105_13168_b200 as dt
import torch
mesh = dt.TriangleMesh.generate(sys.argv[1] if len(sys.argv) > 1 else "genus:8:45")
verts, faces = mesh.vertices(), mesh.faces()
vpin = torch.from_numpy(verts).pin_memory().numpy()
fpin = torch.from_numpy(faces.astype(np.int32)).pin_memory().numpy().view(np.uint32)
for i in range(3):
    m = dt.TriangleMesh.from_arrays(vpin, fpin)
    o = dt.assemble_laplacian(m)
    torch.cuda.synchronize()
    del o, m
