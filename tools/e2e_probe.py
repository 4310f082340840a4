"""e2e stage timing probe (diagnostics, GPU box): DTB_TIMING=1 python tools/e2e_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2105_13168_b200 as dt
import torch
spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
mesh = dt.TriangleMesh.generate(spec)
verts, faces = mesh.vertices(), mesh.faces()
vpin = torch.from_numpy(verts).pin_memory().numpy()
fpin = torch.from_numpy(faces.astype(np.int32)).pin_memory().numpy().view(np.uint32)
cfg = dt.default_config(max_steps=3000)
for i in range(4):
    t0 = time.perf_counter()
    m = dt.TriangleMesh.from_arrays(vpin, fpin)
    t1 = time.perf_counter()
    o = dt.assemble_laplacian(m)
    t2 = time.perf_counter()
    r = dt.run_initial_pass(m, o, 0, cfg)
    t3 = time.perf_counter()
    evs = r.events(); trs = r.tracks()
    t4 = time.perf_counter()
    print(f"rep {i}: mesh {1e3*(t1-t0):.2f} op {1e3*(t2-t1):.2f} pass {1e3*(t3-t2):.2f} (device {1e3*r.timing()['t_pass_device']:.2f}) results {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms", flush=True)
    del r, o, m
