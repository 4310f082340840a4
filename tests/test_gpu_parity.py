"""Device engine vs. the compiled reference (oracle/_ref) on the same inputs.

Bit-exact: stiffness off-diagonals, masses, every field value after every step
(64-bit field digests per check), event logs, loop anchors, covered sets and
estimate snapshots.  Tolerance-bounded: stiffness diagonals (8 ulp, summation
order of the reference's std::sort is not reproducible) and vanish positions
(fixed-point device band means, 1e-9)."""
import numpy as np
import pytest

import paper_2105_13168_b200 as dt
from tests import parity, refdata

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refdata.have_ref(), reason="oracle/_ref not built")]

SMALL = ["icosphere:3:2.0", "torus:32:16:2:0.5", "genus:1:2", "genus:2:2", "torus_irr:32:16:2:0.5:0.3:0.05:7"]


def ref_operator(mesh, spec):
    L = refdata.ref_laplacian(spec)
    return dt.LaplacianOperator.from_csr(mesh, L["off"], L["col"], L["val"], L["mass"], L["gershgorin"]), L


@pytest.mark.parametrize("spec", SMALL + ["limbstar:3:3:4", "coin:8:24:3:1"])
def test_laplacian_assembly(spec):
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    off, col, val, mass = op.csr()
    L = refdata.ref_laplacian(spec)
    assert np.array_equal(off, L["off"]) and np.array_equal(col, L["col"])
    assert np.array_equal(mass.view(np.uint64), L["mass"].view(np.uint64))
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
    diag = rows == col
    assert np.array_equal(val[~diag].view(np.uint64), L["val"][~diag].view(np.uint64))
    ulp = np.abs(val[diag].view(np.int64) - L["val"][diag].view(np.int64))
    assert ulp.max() <= 8, ulp.max()
    assert op.gershgorin_bound == pytest.approx(L["gershgorin"], rel=1e-14)


@pytest.mark.parametrize("spec,steps", [(s, 300) for s in SMALL])
def test_initial_pass_bit_exact(spec, steps):
    mesh = dt.TriangleMesh.generate(spec)
    op, _ = ref_operator(mesh, spec)
    cfg = dt.default_config(max_steps=steps, record_hashes=1)
    res = dt.run_initial_pass(mesh, op, 0, cfg)
    ref = refdata.ref_run(spec, max_steps=steps)
    assert res.status == ("ok" if ref["status"] == "ok" else ref["error_type"])
    assert res.steps == ref["steps"]
    mine = [int(h) for h in res.hashes()]
    theirs = [int(h) for h in ref["hashes"]]
    assert len(mine) == len(theirs)
    first_bad = next((i for i, (a, b) in enumerate(zip(mine, theirs)) if a != b), None)
    assert first_bad is None, f"field digest diverges at check {first_bad + 1}"
    parity.compare_events(res.events(), ref["events"])
    exact, total = parity.compare_tracks(res.tracks(), ref["tracks"])
    # Trail points snap the band mean to its nearest band vertex.  On the
    # symmetric generators whole rings of band vertices tie with the mean up to
    # rounding noise, so which one the reference picks is noise; only the
    # irregular mesh is held to an exact-match rate.
    if spec.startswith("torus_irr"):
        assert total == 0 or exact / total > 0.9, (exact, total)


@pytest.mark.parametrize("spec,steps", [("torus:64:32:2:0.5", 1500), ("genus:2:3", 1500), ("torus:48:24:3:1.2", 2000)])
def test_device_assembled_pass_matches_oracle(spec, steps):
    """End to end on the device-assembled operator: the oracle consumes the same
    operator, so every field digest and event must agree bit for bit."""
    from oracle import oracle as orc
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    off, col, val, mass = op.csr()
    ref = orc.run_initial_pass(spec, steps, operator=(off, col, val, mass, op.gershgorin_bound))
    assert [int(h) for h in res.hashes()] == ref["hashes"]
    parity.compare_events(res.events(), ref["events"])
    parity.compare_tracks(res.tracks(), ref["tracks"])


@pytest.mark.parametrize("spec", ["torus:32:16:2:0.5", "genus:2:2"])
def test_check_interval_and_overrides(spec):
    from oracle import oracle as orc
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=400, record_hashes=1, check_interval=3,
                                                               dt=5.0, collision_threshold=0.2))
    off, col, val, mass = op.csr()
    ref = orc.run_initial_pass(spec, 400, operator=(off, col, val, mass, op.gershgorin_bound), check_interval=3,
                               dt=5.0, kappa=0.2)
    assert [int(h) for h in res.hashes()] == ref["hashes"]
    parity.compare_events(res.events(), ref["events"])


def test_repeated_passes_reuse_workspace():
    mesh = dt.TriangleMesh.generate("torus:32:16:2:0.5")
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=300, record_hashes=1)
    a = dt.run_initial_pass(mesh, op, 0, cfg)
    ha = [int(h) for h in a.hashes()]
    del a
    b = dt.run_initial_pass(mesh, op, 0, cfg)
    assert [int(h) for h in b.hashes()] == ha
    c = dt.run_initial_pass(mesh, op, 7, cfg)  # different seed: different trajectory
    assert [int(h) for h in c.hashes()] != ha


def test_cpp_facade_runs(tmp_path):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "detect_loops"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{root}/include", f"{root}/examples/detect_loops.cpp",
                    f"-L{root}/paper_2105_13168_b200/lib", "-ldifftopo_b200",
                    f"-Wl,-rpath,{root}/paper_2105_13168_b200/lib", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "icosphere:3:2.0"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert '"status":0' in out.stdout and "vanish" in out.stdout and "cycle_rank 0" in out.stdout


def test_event_heavy_chaotic_torus_matches_reference():
    """Hundreds of splits/merges/vanishes (the reference's chaotic regime on a
    coarse torus): the trajectory must stay bit-exact through every event."""
    spec, steps = "torus:96:32:3:1.0", 7000
    mesh = dt.TriangleMesh.generate(spec)
    op, _ = ref_operator(mesh, spec)
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    ref = refdata.ref_run(spec, max_steps=steps)
    assert len(ref["events"]) > 80
    mine, theirs = [int(h) for h in res.hashes()], [int(h) for h in ref["hashes"]]
    first_bad = next((i for i, (a, b) in enumerate(zip(mine, theirs)) if a != b), None)
    assert first_bad is None and len(mine) == len(theirs), first_bad
    parity.compare_events(res.events(), ref["events"])
    parity.compare_tracks(res.tracks(), ref["tracks"])


def test_result_queries_after_pass_and_between_passes():
    """A result keeps its field after the pass engine (and its stream) is gone;
    its device queries must keep working, also after further passes."""
    mesh = dt.TriangleMesh.generate("genus:2:3")
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=500)
    r1 = dt.run_initial_pass(mesh, op, 0, cfg)
    h1 = r1.field_hash()
    r2 = dt.run_initial_pass(mesh, op, 5, cfg)
    assert r1.field_hash() == h1
    assert r2.field_hash() != 0
    v, x = r1.layer_values(1)
    assert len(v) == len(x)


@pytest.mark.parametrize("spec,steps", [("torus:96:32:3:1.0", 2500), ("genus:2:3", 1500)])
def test_split_certificate_matches_full_union_find(spec, steps, monkeypatch):
    """The split certificate (skipping the front union-find on steps that
    cannot split a front) gives the same trajectory and events as running the
    union-find at every check (DTB_D_FULL=1)."""
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=steps, record_hashes=1)
    fast = dt.run_initial_pass(mesh, op, 0, cfg)
    monkeypatch.setenv("DTB_D_FULL", "1")
    full = dt.run_initial_pass(mesh, op, 0, cfg)
    assert [int(h) for h in fast.hashes()] == [int(h) for h in full.hashes()]
    assert [(e.kind, e.step, e.layers) for e in fast.events()] == [(e.kind, e.step, e.layers) for e in full.events()]


@pytest.mark.parametrize("spec,steps", [("torus_irr:40:20:2:0.6:0.2:0.05:7", 800), ("genus:2:3", 600)])
def test_trail_snap_overflow_list_matches_segments(spec, steps, monkeypatch):
    """Band items for the trail snap go to per-CTA segments; a full segment
    spills into the shared overflow list.  Tiny segments (DTB_BP_SEG=3) force
    nearly every item through the overflow path: trails must not change."""
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=steps, record_hashes=1)
    a = dt.run_initial_pass(mesh, op, 0, cfg)
    monkeypatch.setenv("DTB_BP_SEG", "3")
    b = dt.run_initial_pass(mesh, op, 0, cfg)
    assert [int(h) for h in a.hashes()] == [int(h) for h in b.hashes()]
    ta, tb = a.tracks(), b.tracks()
    assert len(ta) == len(tb) and sum(len(t["trail"]) for t in ta) > 0
    for x, y in zip(ta, tb):
        assert x["layer"] == y["layer"]
        np.testing.assert_array_equal(np.asarray(x["trail"]), np.asarray(y["trail"]))


def test_trail_snap_overflow_raises_capacity_error(monkeypatch):
    """When the band items of a check fill both the segments and the overflow
    list, the pass fails with a capacity error instead of snapping trails from
    a truncated list (the stop used to look like an ordinary event)."""
    mesh = dt.TriangleMesh.generate("torus:32:16:2:0.5")
    op = dt.assemble_laplacian(mesh)
    monkeypatch.setenv("DTB_BP_SEG", "1")
    monkeypatch.setenv("DTB_BP_OVF", "2")
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=300))
    assert res.status == "CapacityExceeded"
    assert "band item list overflow" in res.message


@pytest.mark.parametrize("spec,steps", [("torus:48:24:3:1.2", 2000), ("genus:2:3", 1500)])
def test_device_built_mesh_events_match_reference(spec, steps, monkeypatch, capfd):
    """A device-built mesh (from_arrays) has no host copy: its splits, merges,
    vanishes and handle loops are computed from local gathers of the rows,
    faces and edges they touch -- bit-exact with the reference, and without
    downloading the whole mesh."""
    host = dt.TriangleMesh.generate(spec)
    mesh = dt.TriangleMesh.from_arrays(host.vertices(), host.faces())
    op, _ = ref_operator(mesh, spec)
    monkeypatch.setenv("DTB_TIMING", "1")
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    monkeypatch.delenv("DTB_TIMING")
    assert "host mesh download" not in capfd.readouterr().err
    ref = refdata.ref_run(spec, max_steps=steps)
    assert len(ref["events"]) > 5
    mine, theirs = [int(h) for h in res.hashes()], [int(h) for h in ref["hashes"]]
    first_bad = next((i for i, (a, b) in enumerate(zip(mine, theirs)) if a != b), None)
    assert first_bad is None and len(mine) == len(theirs), first_bad
    parity.compare_events(res.events(), ref["events"])
    parity.compare_tracks(res.tracks(), ref["tracks"])


@pytest.mark.parametrize("spec,steps", [("gyroid:2:26:0.3:1.0", 1500), ("gyroid:4:20:0.3:1.0", 400)])
def test_gyroid_wide_columns_bit_exact(spec, steps, tmp_path):
    """High-genus gyroids split the seed front into six layers within a few
    steps, so a third of the frontier carries 5-10 candidate layers and takes
    the lane-parallel wide update (or the sequential general one beyond it):
    field digests and events bit-exact with the reference on the same mesh."""
    host = dt.TriangleMesh.generate(spec)
    path = str(tmp_path / "g.dtm")
    host.save(path)
    ref_spec = "dtm:" + path
    mesh = dt.TriangleMesh.from_arrays(host.vertices(), host.faces())
    op, _ = ref_operator(mesh, ref_spec)
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    ref = refdata.ref_run(ref_spec, max_steps=steps)
    assert len(ref["events"]) >= 2 and len(ref["events"][1]["produced"]) >= 3
    mine, theirs = [int(h) for h in res.hashes()], [int(h) for h in ref["hashes"]]
    first_bad = next((i for i, (a, b) in enumerate(zip(mine, theirs)) if a != b), None)
    assert first_bad is None and len(mine) == len(theirs), first_bad
    parity.compare_events(res.events(), ref["events"])


@pytest.mark.parametrize("spec,steps", [("genus:8:45", 3000), ("genus:4:45", 3000)])
def test_bench_workload_final_state_bit_exact(spec, steps):
    """The bench workload itself (configs[1], V = 988k; configs[3], V = 535k):
    a full 3000-step pass ends in the reference's exact field (64-bit digest
    of every stored value), with the same events and step count."""
    mesh = dt.TriangleMesh.generate(spec)
    op, _ = ref_operator(mesh, spec)
    res = dt.run_initial_pass(mesh, op, 0, dt.default_config(max_steps=steps))
    ref = refdata.ref_run(spec, max_steps=steps)
    assert res.status == ("ok" if ref["status"] == "ok" else ref["error_type"])
    assert res.steps == ref["steps"]
    assert res.field_hash() == int(ref["final_hash"])
    parity.compare_events(res.events(), ref["events"])


@pytest.mark.parametrize("spec,steps,seed", [("genus:8:45", 3000, 0), ("gyroid:2:26:0.3:1.0", 1500, 0),
                                             ("torus:96:32:3:1.0", 2000, 0), ("limbstar:2:3:3", 2000, 0),
                                             ("plate:2:20:0.5", 2000, 0), ("plate:2:20:0.5", 2000, 30000),
                                             ("torus_irr:40:20:2:0.6:0.2:0.05:7", 2000, 11),
                                             ("icosphere:3:2.0", 600, 5), ("genus:2:3", 2000, 100)])
def test_split_certificate_never_hides_a_split(spec, steps, seed, monkeypatch):
    """DTB_CERT_VERIFY=1 runs the union-find after every check whose split
    certificate held (gained items anchored, lost items' stars connected)
    and fails the pass if it finds two components there; the pass must
    finish as the plain one does, in the same field state."""
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=steps)
    plain = dt.run_initial_pass(mesh, op, seed, cfg)
    monkeypatch.setenv("DTB_CERT_VERIFY", "1")
    checked = dt.run_initial_pass(mesh, op, seed, cfg)
    assert checked.status == plain.status and checked.steps == plain.steps
    assert checked.field_hash() == plain.field_hash()
    assert [(e.kind, e.step, e.layers) for e in checked.events()] == [(e.kind, e.step, e.layers)
                                                                       for e in plain.events()]


@pytest.mark.parametrize("spec", ["genus:8:45", "torus_irr:40:20:2:0.6:0.2:0.05:7", "gyroid:2:26:0.3:1.0"])
def test_operator_apply_matches_csr_sums(spec):
    """LaplacianOperator.apply (the padded-row SpMV the sweep benchmark
    times) equals M^-1 S x summed in CSR row order, bit for bit."""
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    off, col, val, mass = op.csr()
    x = np.random.default_rng(3).standard_normal(len(mass))
    y = op.apply(x)
    # Row-order sums, one column of the padded rows at a time (adding +0.0
    # for a missing entry leaves a sum that starts at +0.0 unchanged).
    lens = np.diff(off)
    width = int(lens.max())
    idx = np.minimum(off[:-1, None] + np.arange(width)[None, :], len(col) - 1)
    prod = val[idx] * x[col[idx]]
    acc = np.zeros(len(mass))
    for j in range(width):
        acc = acc + np.where(j < lens, prod[:, j], 0.0)
    assert np.array_equal(y, acc / mass)


def _grid_cube_obj(path, n):
    """Closed cube surface, n x n squares per side, each split along one
    diagonal: every diagonal's two opposite angles are right angles, so its
    cotangent weight is exactly zero (the reference drops it)."""
    index, verts, faces = {}, [], []

    def vid(p):
        if p not in index:
            index[p] = len(verts)
            verts.append(p)
        return index[p]

    for axis in range(3):
        for side in (0, n):
            for i in range(n):
                for j in range(n):
                    quad = []
                    for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        p = [0, 0, 0]
                        p[axis] = side
                        p[(axis + 1) % 3] = i + di
                        p[(axis + 2) % 3] = j + dj
                        quad.append(vid(tuple(p)))
                    a, b, c, d = quad if side == n else quad[::-1]
                    faces += [(a, b, c), (a, c, d)]
    with open(path, "w") as fh:
        for p in verts:
            fh.write("v %d %d %d\n" % p)
        for f in faces:
            fh.write("f %d %d %d\n" % (f[0] + 1, f[1] + 1, f[2] + 1))


def test_laplacian_assembly_drops_exact_zero_weights(tmp_path):
    """Rows with exact zero weights leave the no-count assembly for the
    counted one; the operator matches the reference's entry for entry."""
    path = str(tmp_path / "cube.obj")
    _grid_cube_obj(path, 6)
    spec = "file:" + path
    mesh = dt.TriangleMesh.generate(spec)
    op = dt.assemble_laplacian(mesh)
    off, col, val, mass = op.csr()
    assert np.count_nonzero(val == 0.0) == 0
    assert len(val) < (len(off) - 1) + 2 * mesh.info()["E"]  # zeros were dropped
    L = refdata.ref_laplacian(spec)
    assert np.array_equal(off, L["off"]) and np.array_equal(col, L["col"])
    assert np.array_equal(mass.view(np.uint64), L["mass"].view(np.uint64))
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
    diag = rows == col
    assert np.array_equal(val[~diag].view(np.uint64), L["val"][~diag].view(np.uint64))
