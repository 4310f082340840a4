"""Manual GPU smoke: python -m tests.quick_gpu (not collected by pytest)."""
import sys, time
import numpy as np
import paper_2105_13168_b200 as dt
from tests import refdata, parity

print(dt.device_info(), flush=True)
for spec, steps in [("icosphere:3:2.0", 500), ("torus:32:16:2:0.5", 300), ("genus:1:2", 300)]:
    mesh = dt.TriangleMesh.generate(spec)
    L = refdata.ref_laplacian(spec)
    op = dt.LaplacianOperator.from_csr(mesh, L["off"], L["col"], L["val"], L["mass"], L["gershgorin"])
    t0 = time.time()
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    t1 = time.time()
    ref = refdata.ref_run(spec, max_steps=steps)
    mine = [int(h) for h in res.hashes()]; theirs = [int(h) for h in ref["hashes"]]
    bad = next((i for i, (a, b) in enumerate(zip(mine, theirs)) if a != b), None)
    print(spec, res.status, res.steps, "events", res.n_events, "ref", len(ref["events"]), ref["status"],
          "hash_len", len(mine), len(theirs), "first_bad", bad, "gpu_s", round(t1 - t0, 3), "ref_s", round(ref["seconds"], 3),
          res.timing(), flush=True)
    for a, b in list(zip(res.events(), ref["events"]))[:6]:
        print("   ", a.kind, a.step, a.layers, a.produced, "|", b["kind"], b["step"], b["layers"], b["produced"])
