"""Regenerates the golden fixtures from the compiled reference (oracle/_ref,
built by `make -C oracle ref` from the unmodified /root/reference headers).

    python tests/golden/make_golden.py

Fixtures are compact: per-check 64-bit field digests, full event logs (loops,
covered sets, estimate snapshot digests), track lifetimes with trail digests,
operator and mesh digests.  Only this script reads the reference; tests read
the committed JSON."""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from tests import refdata  # noqa: E402

RUNS = [
    ("icosphere:3:2.0", 500),
    ("torus:32:16:2:0.5", 400),
    ("genus:1:2", 300),
    ("genus:2:2", 300),
    ("torus_irr:32:16:2:0.5:0.3:0.05:7", 300),
    ("torus:16:8:2:0.5", 200),
    ("coin:8:24:3:1", 200),
]
MESHES = ["torus:16:8:2:0.5", "torus:64:32:2:0.5", "genus:2:3", "icosphere:3:2.0", "limbstar:3:3:4",
          "coin:8:24:3:1", "torus_irr:32:16:2:0.5:0.3:0.05:7", "genus:5:2", "genus:0:3"]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def trail_digest(trail):
    return digest(np.asarray(trail, np.float64).reshape(-1, 3)) if len(trail) else ""


def read_dtm_topo(path):
    import struct
    b = open(path, "rb").read()
    nv, nf = struct.unpack_from("<II", b, 4)
    o = 12
    v = np.frombuffer(b, np.float64, 3 * nv, o); o += 24 * nv
    f = np.frombuffer(b, np.uint32, 3 * nf, o); o += 12 * nf
    o += 4
    ne, = struct.unpack_from("<I", b, o); o += 4
    ev = np.frombuffer(b, np.uint32, 2 * ne, o); o += 8 * ne
    ef = np.frombuffer(b, np.uint32, 2 * ne, o); o += 8 * ne
    fe = np.frombuffer(b, np.uint32, 3 * nf, o)
    return v, f, ev, ef, fe


def main():
    meshes = {}
    for spec in MESHES:
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "m.dtm")
            out = subprocess.run([refdata.REF_BIN, "mesh", spec, p], check=True, capture_output=True, text=True)
            info = json.loads(out.stdout)
            v, f, ev, ef, fe = read_dtm_topo(p)
            L = refdata.ref_laplacian(spec)
            meshes[spec] = dict(info, vertices=digest(v), faces=digest(f), edge_vertices=digest(ev),
                                edge_faces=digest(ef), face_edges=digest(fe), csr_off=digest(L["off"]),
                                csr_col=digest(L["col"]), csr_val=digest(L["val"]), mass=digest(L["mass"]),
                                gershgorin=L["gershgorin"], dt=L["dt"])
    runs = {}
    for spec, steps in RUNS:
        r = refdata.ref_run(spec, max_steps=steps)
        runs[f"{spec}@{steps}"] = {
            "status": r["status"], "error_type": r.get("error_type"), "steps": r["steps"], "dt_used": r["dt_used"],
            "hashes": r["hashes"], "events": r["events"],
            "tracks": [{"layer": t["layer"], "created": t["created"], "consumed": t["consumed"],
                        "trail_n": len(t["trail"]), "trail": trail_digest(t["trail"])} for t in r["tracks"]],
        }
    # Isolines of analytic fields (isoline.hpp:55).
    iso = {}
    for spec, level in [("coin:8:24:3:1", 0.5), ("torus:32:16:2:0.5", 0.3), ("genus:2:3", 0.45)]:
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "m.dtm")
            subprocess.run([refdata.REF_BIN, "mesh", spec, p], check=True, capture_output=True)
            v = read_dtm_topo(p)[0].reshape(-1, 3)
        vals = 0.5 + 0.5 * np.sin(1.3 * v[:, 0] + 0.7 * v[:, 1] - 0.4 * v[:, 2])
        loops = refdata.ref_isoline(spec, vals, level)
        iso[f"{spec}@{level}"] = {"field": "0.5+0.5*sin(1.3x+0.7y-0.4z)", "loops": loops}
    # seed_region (diffusion.hpp:134) with the default radius, and one step().
    seeds, steps1 = {}, {}
    for spec in ["torus:32:16:2:0.5", "genus:2:3", "icosphere:3:2.0", "limbstar:3:3:4"]:
        s = refdata.ref_step(spec, n=3)
        seeds[spec] = s["seeds"]
        steps1[spec] = {"n": 3, "hash": s["hash"]}
    out = {"generator": "tests/golden/make_golden.py (oracle/_ref)", "meshes": meshes, "runs": runs, "isolines": iso,
           "seeds": seeds, "one_shot_steps": steps1}
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "reference_fixtures.json"))


if __name__ == "__main__":
    main()
