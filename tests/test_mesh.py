"""Host-side mesh construction, generators and IO of the product (no GPU
needed) against the reference's golden digests (mesh.hpp, generators.hpp,
mesh_io.hpp)."""
import hashlib
import os

import numpy as np
import pytest

import paper_2105_13168_b200 as dt
from tests import refdata

GOLD = refdata.load_golden("reference_fixtures.json")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.mark.parametrize("spec", sorted(GOLD["meshes"]))
def test_generated_mesh_matches_reference(spec):
    g = GOLD["meshes"][spec]
    m = dt.TriangleMesh.generate(spec)
    info = m.info()
    assert (info["V"], info["E"], info["F"], info["genus"]) == (g["V"], g["E"], g["F"], g["genus"])
    assert digest(m.vertices()) == g["vertices"]
    assert digest(m.faces()) == g["faces"]
    ev, ef = m.edges()
    assert digest(ev) == g["edge_vertices"]
    assert digest(ef) == g["edge_faces"]
    assert digest(m.face_edges()) == g["face_edges"]


@pytest.mark.parametrize("g", [0, 1, 2, 3, 5, 6])
def test_genus_of_generated_surfaces(g):
    assert dt.TriangleMesh.generate(f"genus:{g}:2").info()["genus"] == g


def test_torus_counts():
    info = dt.TriangleMesh.generate("torus:16:8:2:0.5").info()
    assert (info["V"], info["F"], info["E"], info["genus"]) == (128, 256, 384, 1)
    assert dt.TriangleMesh.generate("torus:3:3:2:0.5").info()["genus"] == 1


def test_invalid_parameters():
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.generate("torus:16:8:2:2.1")
    assert e.value.kind == "InvalidParameter"


def _icosahedron():
    m = dt.TriangleMesh.generate("icosphere:0:1.0")
    return m.vertices(), m.faces()


def test_validation_rejects_open_and_broken_meshes():
    v, f = _icosahedron()
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v, f[:-1])  # one face removed: boundary edges
    assert e.value.kind == "TopologyError"
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v[:3], np.array([[0, 1, 2]]))
    assert e.value.kind == "TopologyError"
    bad = f.copy()
    bad[0] = [bad[0][0], bad[0][0], bad[0][1]]
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v, bad)
    assert e.value.kind == "DegeneracyError"
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v, np.vstack([f, f[:1]]))
    assert e.value.kind == "TopologyError"
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v, np.where(f == 0, 99, f))
    assert e.value.kind == "ParseError"
    # Two disjoint icosahedra: multiple components.
    v2 = np.vstack([v, v + 10.0])
    f2 = np.vstack([f, f + len(v)])
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.from_arrays(v2, f2)
    assert e.value.kind == "TopologyError"


def test_orientation_is_normalised():
    v, f = _icosahedron()
    flipped = f.copy()
    flipped[:, [1, 2]] = flipped[:, [2, 1]]
    flipped[3, [1, 2]] = flipped[3, [2, 1]]  # one face inconsistent with the rest
    m = dt.TriangleMesh.from_arrays(v, flipped)
    assert np.array_equal(m.faces(), f)


def test_unreferenced_vertices_dropped():
    v, f = _icosahedron()
    v2 = np.vstack([[[9.0, 9.0, 9.0]], v])
    m = dt.TriangleMesh.from_arrays(v2, f + 1)
    assert m.info()["V"] == 12


def test_io_round_trip(tmp_path):
    m = dt.TriangleMesh.generate("genus:2:2")
    for ext in ("ply", "obj", "dtm"):
        p = str(tmp_path / f"m.{ext}")
        m.save(p)
        m2 = dt.TriangleMesh.load(p)
        assert m2.info() == m.info()
        assert np.array_equal(m2.faces(), m.faces())
        assert np.allclose(m2.vertices(), m.vertices(), rtol=0, atol=1e-12)
    off = tmp_path / "ico.off"
    v, f = _icosahedron()
    with open(off, "w") as fh:
        fh.write("OFF\n# comment\n12 20 30\n")
        for p in v:
            fh.write(f"{float(p[0])!r} {float(p[1])!r} {float(p[2])!r}\n")
        for t in f:
            fh.write(f"3 {t[0]} {t[1]} {t[2]}\n")
    m3 = dt.TriangleMesh.load(str(off))
    assert m3.info()["V"] == 12 and m3.info()["E"] == 30 and m3.info()["genus"] == 0


def test_parse_errors(tmp_path):
    p = tmp_path / "bad.off"
    p.write_text("OFF\n3 1 0\n0 0 0\n1 0 0\n")
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.load(str(p))
    assert e.value.kind == "ParseError"
    q = tmp_path / "tri.obj"
    q.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    with pytest.raises(dt.DiffTopoError) as e:
        dt.TriangleMesh.load(str(q))
    assert e.value.kind == "TopologyError"


@pytest.mark.parametrize("spec", sorted(GOLD["seeds"]))
def test_seed_region_matches_reference(spec):
    m = dt.TriangleMesh.generate(spec)
    s = m.seed_region(0, 1.5 * (1 / 25) / np.sqrt(1 / 125))
    assert s.tolist() == GOLD["seeds"][spec]
