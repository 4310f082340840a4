"""Per-phase step profile of the engine (manual; GPU box):

    DTB_PHASE_PROF=1 python tools/phase_prof.py [spec] [steps]

prints the engine's '[dtb] phase us/step' line (stderr) for one pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
m = dt.TriangleMesh.generate(spec)
op = dt.assemble_laplacian(m)
for _ in range(2):
    r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=steps))
    print(spec, r.status, r.steps, len(r.events()), f"{1e3 * r.timing()['t_pass_device']:.2f} ms", flush=True)
