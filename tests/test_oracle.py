"""The CPU restatement (oracle/difftopo_oracle.cpp) against the reference's
golden fixtures (tests/golden/reference_fixtures.json, generated from the
compiled reference by tests/golden/make_golden.py) and, when oracle/_ref is
built, against the reference itself on longer horizons."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from tests import refdata

GOLD = refdata.load_golden("reference_fixtures.json")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def trail_digest(trail):
    return digest(np.asarray(trail, np.float64).reshape(-1, 3)) if len(trail) else ""


@pytest.mark.parametrize("key", sorted(GOLD["runs"]))
def test_oracle_matches_golden_run(key):
    spec, steps = key.rsplit("@", 1)
    g = GOLD["runs"][key]
    o = orc.run_initial_pass(spec, int(steps))
    assert o["status"] == g["status"] and o.get("error_type") == g["error_type"]
    assert o["steps"] == g["steps"]
    assert o["dt_used"] == g["dt_used"]
    assert o["hashes"] == [int(h) for h in g["hashes"]]
    assert o["events"] == g["events"]
    got = [{"layer": t["layer"], "created": t["created"], "consumed": t["consumed"], "trail_n": len(t["trail"]),
            "trail": trail_digest(t["trail"])} for t in o["tracks"]]
    assert got == g["tracks"]


@pytest.mark.parametrize("spec", sorted(GOLD["meshes"]))
def test_oracle_assembly_matches_golden(spec):
    g = GOLD["meshes"][spec]
    L = orc.assemble(spec)
    assert digest(L["off"].astype(np.int64)) == g["csr_off"]
    assert digest(L["col"].astype(np.int64)) == g["csr_col"]
    assert digest(L["val"]) == g["csr_val"]
    assert digest(L["mass"]) == g["mass"]
    assert L["gershgorin"] == g["gershgorin"]


@pytest.mark.skipif(not refdata.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("spec,steps", [("torus:32:16:2:0.5", 1500), ("genus:2:2", 1200),
                                        ("torus:48:24:3:1.2", 600), ("limbstar:2:3:3", 600)])
def test_oracle_matches_reference_long(spec, steps):
    o = orc.run_initial_pass(spec, steps)
    r = refdata.ref_run(spec, max_steps=steps)
    assert o["hashes"] == [int(h) for h in r["hashes"]]
    assert o["events"] == r["events"]
    assert [(t["layer"], t["created"], t["consumed"], t["trail"]) for t in o["tracks"]] == \
           [(t["layer"], t["created"], t["consumed"], t["trail"]) for t in r["tracks"]]


def test_oracle_config_overrides():
    # check_interval > 1 and an explicit dt take the reference's code paths too.
    if not refdata.have_ref():
        pytest.skip("oracle/_ref not built")
    o = orc.run_initial_pass("torus:32:16:2:0.5", 300, check_interval=3, dt=5.0, kappa=0.2)
    r = refdata.ref_run("torus:32:16:2:0.5", max_steps=300, check_interval=3, dt=5.0, kappa=0.2)
    assert o["hashes"] == [int(h) for h in r["hashes"]]
    assert o["events"] == r["events"]
