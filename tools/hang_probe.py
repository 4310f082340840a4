"""One pass with progress (diagnostics): python tools/hang_probe.py spec steps"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt
spec, steps = sys.argv[1], int(sys.argv[2])
m = dt.TriangleMesh.generate(spec)
op = dt.assemble_laplacian(m)
print("start", flush=True)
t = time.time()
r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
print(spec, r.status, r.steps, len(r.events()), f"{time.time() - t:.2f}s", flush=True)
