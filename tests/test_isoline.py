"""extract_isoline (isoline.hpp:55) of the product's host path against the
reference's golden loops."""
import numpy as np
import pytest

import paper_2105_13168_b200 as dt
from tests import refdata

GOLD = refdata.load_golden("reference_fixtures.json")


@pytest.mark.parametrize("key", sorted(GOLD["isolines"]))
def test_isoline_matches_reference(key):
    spec, level = key.rsplit("@", 1)
    m = dt.TriangleMesh.generate(spec)
    v = m.vertices()
    vals = 0.5 + 0.5 * np.sin(1.3 * v[:, 0] + 0.7 * v[:, 1] - 0.4 * v[:, 2])
    loops = dt.extract_isoline(m, vals, float(level))
    ref = GOLD["isolines"][key]["loops"]
    assert len(loops) == len(ref)
    for a, b in zip(loops, ref):
        assert [(p.edge, p.t, p.face, tuple(p.position)) for p in a] == [(q[0], q[1], q[2], tuple(q[3])) for q in b]


def test_isoline_empty_and_closed():
    m = dt.TriangleMesh.generate("coin:8:24:3:1")
    assert dt.extract_isoline(m, np.zeros(m.info()["V"]), 0.5) == []
    v = m.vertices()
    r = np.sqrt(v[:, 0] ** 2 + v[:, 1] ** 2)
    loops = dt.extract_isoline(m, r, 1.5)
    assert len(loops) == 2  # top and bottom disk
    for lp in loops:
        assert lp[0].edge == lp[-1].edge and lp[0].t == lp[-1].t
        length = sum(np.linalg.norm(np.subtract(lp[i].position, lp[i + 1].position)) for i in range(len(lp) - 1))
        assert abs(length - 2 * np.pi * 1.5) / (2 * np.pi * 1.5) < 0.05  # analytic circle
