"""Cold-process stage times of one configs[2] e2e call (manual, GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "gyroid:8:26:0.3:1.0"
m0 = dt.TriangleMesh.generate(spec)
v, f = m0.vertices(), m0.faces()
t = [time.perf_counter()]
dt.device_info()
t.append(time.perf_counter())
dt.warmup()
t.append(time.perf_counter())
m = dt.TriangleMesh.from_arrays(v, f)
t.append(time.perf_counter())
op = dt.assemble_laplacian(m)
t.append(time.perf_counter())
r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=3000))
t.append(time.perf_counter())
evs = r.events()
t.append(time.perf_counter())
reeb = r.reeb()
t.append(time.perf_counter())
names = ["device_info", "warmup", "from_arrays", "assemble", "pass", "events", "reeb"]
print({n: round(1e3 * (b - a), 1) for n, a, b in zip(names, t, t[1:])}, r.timing()["t_pass_device"])
