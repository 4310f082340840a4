"""Batch of independent passes (dtb_run_initial_pass_batch, BASELINE
configs[4]): several persistent passes run at once on disjoint SM shares, and
every item must equal its own run_initial_pass -- bit for bit against the
compiled reference where it is cheap, and against the one-at-a-time device run
otherwise.  A failing item reports its own code without disturbing the rest."""
import pytest

import paper_2105_13168_b200 as dt
from paper_2105_13168_b200 import shard
from tests import parity, refdata

pytestmark = pytest.mark.gpu


def _ref_op(mesh, spec):
    L = refdata.ref_laplacian(spec)
    return dt.LaplacianOperator.from_csr(mesh, L["off"], L["col"], L["val"], L["mass"], L["gershgorin"])


@pytest.mark.skipif(not refdata.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("lanes", [1, 3, 8])
def test_batch_items_match_reference(lanes):
    specs = ["torus:32:16:2:0.5", "genus:2:2", "torus_irr:32:16:2:0.5:0.3:0.05:7", "genus:1:2", "icosphere:3:2.0"]
    steps = 600
    meshes = [dt.TriangleMesh.generate(s) for s in specs]
    ops = [_ref_op(m, s) for m, s in zip(meshes, specs)]
    res = dt.run_initial_pass_batch(meshes, ops, None, dt.default_config(max_steps=steps, record_hashes=1),
                                    concurrency=lanes)
    for spec, r in zip(specs, res):
        ref = refdata.ref_run(spec, max_steps=steps)
        assert r.status == ("ok" if ref["status"] == "ok" else ref["error_type"]), spec
        assert r.steps == ref["steps"], spec
        mine, theirs = [int(h) for h in r.hashes()], [int(h) for h in ref["hashes"]]
        assert mine == theirs, spec
        parity.compare_events(r.events(), ref["events"])


def test_batch_equals_sequential_on_configs4_shapes():
    specs = shard.batch_specs(12, 32, 3)[::3]  # genus 1, 4, 7, 10 at the configs[4] resolution
    steps = 800
    meshes = [dt.TriangleMesh.generate(s) for s in specs]
    ops = [dt.assemble_laplacian(m) for m in meshes]
    cfg = dt.default_config(max_steps=steps, record_hashes=1)
    seq = [dt.run_initial_pass(m, o, 0, cfg) for m, o in zip(meshes, ops)]
    for ctas in (0, 5):
        res = dt.run_initial_pass_batch(meshes, ops, [0] * len(specs),
                                        dt.default_config(max_steps=steps, record_hashes=1, grid_ctas=ctas),
                                        concurrency=4)
        for s, a, b in zip(specs, seq, res):
            assert [int(h) for h in a.hashes()] == [int(h) for h in b.hashes()], (s, ctas)
            assert [(e.kind, e.step, e.layers) for e in a.events(with_covered=False)] == \
                   [(e.kind, e.step, e.layers) for e in b.events(with_covered=False)], (s, ctas)


def test_batch_failing_item_is_isolated():
    meshes = [dt.TriangleMesh.generate("torus:32:16:2:0.5") for _ in range(3)]
    ops = [dt.assemble_laplacian(m) for m in meshes]
    cfg = dt.default_config(max_steps=200)
    with pytest.raises(dt.DiffTopoError) as e:
        dt.run_initial_pass_batch(meshes, ops, [0, 10 ** 6, 5], cfg, concurrency=2)
    assert "batch item 1" in str(e.value)
    assert dt.run_initial_pass_batch([], [], None, cfg) == []


def test_cpp_facade_batch(tmp_path):
    import json
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "batch_passes"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{root}/include", f"{root}/examples/batch_passes.cpp",
                    f"-L{root}/paper_2105_13168_b200/lib", "-ldifftopo_b200",
                    f"-Wl,-rpath,{root}/paper_2105_13168_b200/lib", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "4", "300"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    rows = [json.loads(line) for line in out.stdout.splitlines()]
    cfg = dt.default_config(max_steps=300)
    for i, row in enumerate(rows):
        m = dt.TriangleMesh.generate(f"genus:{1 + i}:3")
        r = dt.run_initial_pass(m, dt.assemble_laplacian(m), 0, cfg)
        assert (row["steps"], row["events"]) == (r.steps, r.n_events), i
    assert len(rows) == 4
