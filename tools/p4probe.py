import time, os, sys
sys.path.insert(0, os.getcwd())
import paper_2105_13168_b200 as dt
from paper_2105_13168_b200 import shard
specs = shard.batch_specs(64, 32, 3)
arr = {}
for s in specs:
    m = dt.TriangleMesh.generate(s); arr[s] = (m.vertices(), m.faces())
for mode in ["arrays", "generate", "arrays"]:
    t0 = time.perf_counter()
    ms = [dt.TriangleMesh.from_arrays(*arr[s]) if mode == "arrays" else dt.TriangleMesh.generate(s) for s in specs]
    t1 = time.perf_counter()
    ops = [dt.assemble_laplacian(m) for m in ms]
    t2 = time.perf_counter()
    res = dt.run_initial_pass_batch(ms, ops, None, dt.default_config(max_steps=3000))
    t3 = time.perf_counter()
    tp = sum(r.timing()["t_pass_device"] for r in res)
    print(mode, f"mesh {t1-t0:.3f} ops {t2-t1:.3f} batch {t3-t2:.3f} sum_pass {tp:.3f}", flush=True)
    del res, ops, ms
m = dt.TriangleMesh.from_arrays(*arr[specs[20]]); op = dt.assemble_laplacian(m)
os.environ["DTB_TIMING"] = "1"
r = dt.run_initial_pass(m, op, 0, dt.default_config(max_steps=3000))
print(r.timing())
