"""Manual exploration of workloads on the GPU (not collected by pytest)."""
import sys, time
import paper_2105_13168_b200 as dt

specs = sys.argv[1:] or ["genus:8:45", "plate:8:45:6.0"]
for item in specs:
    spec, steps = (item.split("@") + ["3000"])[:2]
    t0 = time.time(); mesh = dt.TriangleMesh.generate(spec); t1 = time.time()
    op = dt.assemble_laplacian(mesh); t2 = time.time()
    cfg = dt.default_config(max_steps=int(steps))
    res = dt.run_initial_pass(mesh, op, 0, cfg); t3 = time.time()
    info = mesh.info(); tm = res.timing()
    kinds = {}
    for e in res.events(with_covered=False):
        kinds[e.kind] = kinds.get(e.kind, 0) + 1
    print(f"{spec} V={info['V']} genus={info['genus']} gen={t1-t0:.2f}s assemble={t2-t1:.3f}s pass={t3-t2:.3f}s "
          f"status={res.status} steps={res.steps} dt={res.dt_used:.4g} events={kinds} layers={res.layer_count} "
          f"us/step={1e6*(t3-t2)/max(1,res.steps):.1f} avg_region={tm['sum_region']/max(1,res.steps):.0f} "
          f"avg_band={tm['sum_interest']/max(1,res.steps):.0f} {tm}", flush=True)
