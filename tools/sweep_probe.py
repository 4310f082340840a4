"""Full-mesh operator sweep (LaplacianOperator.sweep_bench) for ncu captures
(manual, GPU box):  python tools/sweep_probe.py [spec] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_13168_b200 as dt  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "genus:8:45"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m = dt.TriangleMesh.generate(spec)
op = dt.assemble_laplacian(m)
print(spec, op.sweep_bench(reps))
