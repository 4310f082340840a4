import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2105_13168_b200 as dt
dt.init_work_queues(32)
dt.warmup()
for spec in ["genus:4:45", "genus:4:45"]:
    m0 = dt.TriangleMesh.generate(spec)
    v, f = m0.vertices(), m0.faces()
    t0 = time.perf_counter()
    m = dt.TriangleMesh.from_arrays(v, f)
    t1 = time.perf_counter()
    op = dt.assemble_laplacian(m)
    t2 = time.perf_counter()
    r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=3000))
    t3 = time.perf_counter()
    print(spec, f"mesh {1e3*(t1-t0):.1f} op {1e3*(t2-t1):.1f} pass {1e3*(t3-t2):.1f} ms", r.timing(), flush=True)
