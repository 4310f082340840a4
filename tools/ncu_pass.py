"""One initial pass for ncu captures (manual, GPU box):

    python tools/ncu_pass.py [spec] [steps]

runs run_initial_pass once (the mesh is built and assembled first, so the
engine launch is the only k_engine<0> launch of the process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
m = dt.TriangleMesh.generate(spec)
op = dt.assemble_laplacian(m)
r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=steps))
print(spec, r.status, r.steps, len(r.events()), f"{1e3 * r.timing()['t_pass_device']:.2f} ms", flush=True)
