"""Manual: time the stages of the end-to-end path (not collected by pytest)."""
import sys, time
import numpy as np
import paper_2105_13168_b200 as dt

spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
m0 = dt.TriangleMesh.generate(spec)
v, f = m0.vertices(), m0.faces()
dt.device_info()
for it in range(3):
    t0 = time.perf_counter(); m = dt.TriangleMesh.from_arrays(v, f)
    t1 = time.perf_counter(); db = m.device_bytes()
    t2 = time.perf_counter(); op = dt.assemble_laplacian(m)
    t3 = time.perf_counter(); r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=steps))
    t4 = time.perf_counter(); ev = r.events(); tr = r.tracks()
    t5 = time.perf_counter()
    print(f"mesh {1e3*(t1-t0):.1f} ms  devmesh {1e3*(t2-t1):.1f}  assemble {1e3*(t3-t2):.1f}  pass {1e3*(t4-t3):.1f}  "
          f"results {1e3*(t5-t4):.1f}  total {1e3*(t5-t0):.1f}", flush=True)
    del r, op, m
