"""configs[4] probe (manual, GPU box): the 64-mesh batch run one pass at a
time versus dtb_run_initial_pass_batch at several concurrencies; every batch
item's field digest, status and step count must equal the sequential run's.

    python tools/batch_probe.py [--steps 3000] [--lanes 4,8,16,32]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt  # noqa: E402
from paper_2105_13168_b200 import shard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--lanes", default="4,8,16,32")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--ctas", default="0", help="grid CTAs per pass (0: SMs / lanes)")
    a = ap.parse_args()
    dt.init_work_queues(32)  # opt-in, before any CUDA use
    specs = shard.batch_specs(a.n, 32, 3)
    meshes = [dt.TriangleMesh.generate(s) for s in specs]
    ops = [dt.assemble_laplacian(m) for m in meshes]
    cfg = dt.default_config(max_steps=a.steps)
    dt.run_initial_pass(meshes[0], ops[0], 0, cfg)  # warm-up
    t_cold = None
    for rep in range(2):  # the first round allocates each mesh's workspace
        t0 = time.perf_counter()
        sig, tms = [], []
        for m, o in zip(meshes, ops):  # a caller's loop: each result is dropped after use
            r = dt.run_initial_pass(m, o, 0, cfg)
            sig.append((r.field_hash(), r.status, r.steps, r.n_events))
            tms.append(r.timing())
            del r
        t_seq = time.perf_counter() - t0
        t_cold = t_cold or t_seq
    print(json.dumps({"sequential_cold_s": t_cold}), flush=True)
    print(json.dumps({k: sum(t[k] for t in tms) for k in tms[0] if isinstance(tms[0][k], (int, float))}), flush=True)
    print(json.dumps({"mode": "sequential", "wall_s": t_seq, "meshes": len(specs),
                      "vertices": sum(m.info()["V"] for m in meshes)}), flush=True)
    print(json.dumps({"host_cpus": os.cpu_count(), "sched_cpus": len(os.sched_getaffinity(0))}), flush=True)
    for lanes, ctas in [(int(x), int(c)) for x in a.lanes.split(",") for c in a.ctas.split(",")]:
        bcfg = dt.default_config(max_steps=a.steps, grid_ctas=ctas)
        for rep in range(2):
            t0 = time.perf_counter()
            res = dt.run_initial_pass_batch(meshes, ops, None, bcfg, concurrency=lanes)
            t = time.perf_counter() - t0
            bad = [i for i, r in enumerate(res) if (r.field_hash(), r.status, r.steps, r.n_events) != sig[i]]
            print(json.dumps({"mode": "batch", "lanes": lanes, "ctas": ctas, "rep": rep, "wall_s": t, "speedup": t_seq / t,
                              "mismatches": bad}), flush=True)
            del res


if __name__ == "__main__":
    main()
