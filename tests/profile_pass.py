"""One warm-up pass plus one profiled pass of the bench workload (manual; not
collected by pytest).  Usage: python -m tests.profile_pass [spec] [steps]"""
import sys
import time

import paper_2105_13168_b200 as dt

spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
mesh = dt.TriangleMesh.generate(spec)
op = dt.assemble_laplacian(mesh)
cfg = dt.default_config(max_steps=steps)
for i in range(2):
    t0 = time.time()
    r = dt.run_initial_pass(mesh, op, 0, cfg)
    tm = r.timing()
    print(f"pass {i}: {time.time() - t0:.4f}s status={r.status} {tm}", flush=True)
    del r
