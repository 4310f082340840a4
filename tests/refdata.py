"""Test helpers: run the compiled reference (oracle/_ref/difftopo_ref, built
from the unmodified reference headers by oracle/Makefile) and parse its
outputs.  TEST INFRASTRUCTURE ONLY."""
import json
import os
import struct
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "difftopo_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def have_ref():
    return os.path.exists(REF_BIN)


def ref_run(spec, **kv):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "run.json")
        args = [REF_BIN, "run", spec, out] + [f"{k}={v}" for k, v in kv.items()]
        subprocess.run(args, check=True, capture_output=True)
        with open(out) as f:
            return json.load(f)


def ref_laplacian(spec):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "lap.bin")
        subprocess.run([REF_BIN, "laplacian", spec, out], check=True, capture_output=True)
        return read_laplacian(open(out, "rb").read())


def read_laplacian(b):
    n, = struct.unpack_from("<I", b, 0)
    nnz, = struct.unpack_from("<Q", b, 4)
    o = 12
    off = np.frombuffer(b, np.uint64, n + 1, o).astype(np.int64); o += 8 * (n + 1)
    col = np.frombuffer(b, np.uint32, nnz, o).astype(np.int64); o += 4 * nnz
    val = np.frombuffer(b, np.float64, nnz, o).copy(); o += 8 * nnz
    mass = np.frombuffer(b, np.float64, n, o).copy(); o += 8 * n
    gersh, dt = struct.unpack_from("<dd", b, o)
    return {"off": off, "col": col, "val": val, "mass": mass, "gershgorin": gersh, "dt": dt}


def ref_front(spec, at, **kv):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "front.json")
        subprocess.run([REF_BIN, "front", spec, out, f"at={at}"] + [f"{k}={v}" for k, v in kv.items()],
                       check=True, capture_output=True)
        return json.load(open(out))


def ref_step(spec, n=1, **kv):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "step.json")
        subprocess.run([REF_BIN, "step", spec, out, f"n={n}"] + [f"{k}={v}" for k, v in kv.items()],
                       check=True, capture_output=True)
        j = json.load(open(out))
        j["field"] = read_field_bin(open(out + ".bin", "rb").read())
        return j


def read_field_bin(b):
    lc, V = struct.unpack_from("<II", b, 0)
    o = 8
    layers = []
    for _ in range(lc):
        n, = struct.unpack_from("<I", b, o); o += 4
        rec = np.frombuffer(b, np.dtype([("v", "<u4"), ("x", "<f8")]), n, o); o += 12 * n
        layers.append((rec["v"].copy(), rec["x"].copy()))
    return layers


def ref_isoline(spec, values, level):
    with tempfile.TemporaryDirectory() as d:
        vp = os.path.join(d, "v.f64")
        np.ascontiguousarray(values, np.float64).tofile(vp)
        out = os.path.join(d, "iso.json")
        subprocess.run([REF_BIN, "isoline", spec, vp, repr(float(level)), out], check=True, capture_output=True)
        return json.load(open(out))["loops"]


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)
