"""Device mesh construction (csrc/meshbuild.cu) against the host construction
(csrc/mesh.cpp, the reference's numbering, mesh.hpp:150-324).

`TriangleMesh.from_arrays` builds on the device when a GPU is present and
falls back to the host for unusual or invalid soups; DTB_HOST_MESH=1 forces
the host path.  Every index array must be identical, and invalid soups must
raise the host's errors."""
import os

import numpy as np
import pytest

import paper_2105_13168_b200 as dt
from tests import refdata

pytestmark = pytest.mark.gpu

SPECS = ["torus:32:16:2:0.5", "genus:2:3", "icosphere:3:2.0", "torus_irr:40:20:2:0.6:0.2:0.05:7",
         "limbstar:3:3:4", "coin:8:24:3:1", "genus:8:20", "gyroid:2:8:0.3:1.0"]


def host_built(v, f):
    os.environ["DTB_HOST_MESH"] = "1"
    try:
        return dt.TriangleMesh.from_arrays(v, f)
    finally:
        del os.environ["DTB_HOST_MESH"]


def arrays(m):
    return [m.vertices(), m.faces(), *m.edges(), m.face_edges(), *m.adjacency()]


def assert_same(a, b):
    ia, ib = a.info(), b.info()
    assert ia == ib
    for x, y in zip(arrays(a), arrays(b)):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("spec", SPECS)
def test_device_build_matches_host(spec):
    ref = dt.TriangleMesh.generate(spec)
    v, f = ref.vertices(), ref.faces()
    dev = dt.TriangleMesh.from_arrays(v, f)
    assert_same(dev, ref)


@pytest.mark.parametrize("spec", ["torus:32:16:2:0.5", "genus:3:3"])
def test_device_build_flips_inward_soup(spec):
    ref = dt.TriangleMesh.generate(spec)
    v, f = ref.vertices(), ref.faces()[:, [0, 2, 1]].copy()
    dev = dt.TriangleMesh.from_arrays(v, f)
    assert_same(dev, host_built(v, f))


def test_device_build_shuffled_faces_and_rotated_corners():
    ref = dt.TriangleMesh.generate("genus:2:3")
    v, f = ref.vertices(), ref.faces()
    rng = np.random.default_rng(3)
    f = f[rng.permutation(len(f))]
    f = np.stack([np.roll(row, int(r)) for row, r in zip(f, rng.integers(0, 3, len(f)))])
    assert_same(dt.TriangleMesh.from_arrays(v, f), host_built(v, f))


def test_fallbacks_raise_host_errors():
    ref = dt.TriangleMesh.generate("torus:16:8:2:0.5")
    v, f = ref.vertices(), ref.faces()
    cases = {
        "open": (v, f[:-1]),
        "out of range": (v, np.vstack([f, [[0, 1, len(v) + 5]]]).astype(np.uint32)),
        "out of range, even": (v, np.vstack([f, [[0, 1, len(v) + 5], [1, 0, len(v) + 7]]]).astype(np.uint32)),
        "edge in four faces": (v, np.vstack([f, f[:2]]).astype(np.uint32)),
        "hole and extra": (v, np.vstack([f[2:], [[0, 1, 2], [2, 1, 3]]]).astype(np.uint32)),
    }
    for name, (vv, ff) in cases.items():
        with pytest.raises(dt.DiffTopoError) as dev_err:
            dt.TriangleMesh.from_arrays(vv, ff)
        with pytest.raises(dt.DiffTopoError) as host_err:
            host_built(vv, ff)
        assert str(dev_err.value) == str(host_err.value), name
    # one face flipped: the host re-orients by breadth-first search
    ff = np.vstack([f[:1, [0, 2, 1]], f[1:]]).astype(np.uint32)
    assert_same(dt.TriangleMesh.from_arrays(v, ff), host_built(v, ff))
    # unused vertex: dropped and renumbered by first use (host path)
    vv = np.vstack([v[:1] * 0 + 9.0, v])
    ff = (f + 1).astype(np.uint32)
    assert_same(dt.TriangleMesh.from_arrays(vv, ff), host_built(vv, ff))


@pytest.mark.parametrize("spec,steps", [("genus:2:3", 300), ("torus:32:16:2:0.5", 300)])
def test_pass_on_device_built_mesh_matches_reference(spec, steps):
    ref_mesh = dt.TriangleMesh.generate(spec)
    dev = dt.TriangleMesh.from_arrays(ref_mesh.vertices(), ref_mesh.faces())
    L = refdata.ref_laplacian(spec)
    op = dt.LaplacianOperator.from_csr(dev, L["off"], L["col"], L["val"], L["mass"], L["gershgorin"])
    res = dt.run_initial_pass(dev, op, 0, dt.default_config(max_steps=steps, record_hashes=1))
    ref = refdata.ref_run(spec, max_steps=steps)
    assert [int(h) for h in res.hashes()] == [int(h) for h in ref["hashes"]]
    assert len(res.events()) == len(ref["events"])


@pytest.mark.parametrize("spec", ["torus:32:16:2:0.5", "genus:2:3", "icosphere:3:2.0"])
def test_device_seed_region_matches_host(spec):
    m = dt.TriangleMesh.generate(spec)
    V = m.info()["V"]
    rng = np.random.default_rng(5)
    radii = [0.0, 0.05, 0.3, 0.8]
    for seed in [0, V - 1, *rng.integers(0, V, 4).tolist()]:
        for r in radii:
            host = m.seed_region(int(seed), r)
            os.environ["DTB_SEED_DEVICE"] = "1"
            try:
                dev = m.seed_region(int(seed), r)
            finally:
                del os.environ["DTB_SEED_DEVICE"]
            np.testing.assert_array_equal(dev, host)


def test_device_seed_region_large_matches_host():
    """The bench mesh (V = 988k) at the default seed radius and at a radius
    whose region holds tens of thousands of vertices (wide frontiers)."""
    m = dt.TriangleMesh.generate("genus:8:45")
    for seed, r in [(0, 0.6708203932499369), (12345, 1.5), (987000, 0.2)]:
        host = m.seed_region(seed, r)
        os.environ["DTB_SEED_DEVICE"] = "1"
        try:
            dev = m.seed_region(seed, r)
        finally:
            del os.environ["DTB_SEED_DEVICE"]
        assert len(host) > 0
        np.testing.assert_array_equal(dev, host)
