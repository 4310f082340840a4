"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU restatement
(oracle/difftopo_oracle.cpp -> oracle/build/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker.  Parity of the restatement itself is
pinned against the compiled reference (oracle/_ref) and tests/golden/.
"""
import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: make -C oracle oracle")
        L = C.CDLL(LIB)
        pD, pU, pI = C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_int32)
        L.orc_run.restype = C.c_void_p
        L.orc_run.argtypes = [pD, C.c_uint32, pU, C.c_uint32, pI, pI, pD, pD, C.c_double, C.c_uint32, pD]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_assemble.restype = C.c_long
        L.orc_assemble.argtypes = [pD, C.c_uint32, pU, C.c_uint32, pI, pI, pD, pD, pD]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _mesh_arrays(mesh):
    if isinstance(mesh, str):
        import paper_2105_13168_b200 as dt  # generator verified bit-exact against the reference
        m = dt.TriangleMesh.generate(mesh)
        return m.vertices(), m.faces()
    v, f = mesh
    return np.ascontiguousarray(v, np.float64), np.ascontiguousarray(f, np.uint32)


def assemble(mesh):
    v, f = _mesh_arrays(mesh)
    L = lib()
    nv, nf = len(v), len(f)
    nnz = L.orc_assemble(_p(v, C.c_double), nv, _p(f, C.c_uint32), nf, None, None, None, None, None)
    off = np.empty(nv + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    mass = np.empty(nv, np.float64)
    g = C.c_double()
    L.orc_assemble(_p(v, C.c_double), nv, _p(f, C.c_uint32), nf, _p(off, C.c_int32), _p(col, C.c_int32),
                   _p(val, C.c_double), _p(mass, C.c_double), C.byref(g))
    return {"off": off, "col": col, "val": val, "mass": mass, "gershgorin": g.value}


def run_initial_pass(mesh, max_steps, operator=None, seed=0, dt=0.0, band=0.05, sat=0.999, kappa=0.1,
                     check_interval=1, covered=0.05, seed_radius=0.0, trails=True):
    """Returns the reference driver's JSON structure; hashes as Python ints."""
    v, f = _mesh_arrays(mesh)
    L = lib()
    cfg = np.array([dt, band, sat, kappa, check_interval, max_steps, covered, seed_radius, 1.0 if trails else 0.0],
                   np.float64)
    keep = []
    if operator is not None:
        off, col, val, mass, g = operator
        off = np.ascontiguousarray(off, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        mass = np.ascontiguousarray(mass, np.float64)
        keep = [off, col, val, mass]
        args = (_p(off, C.c_int32), _p(col, C.c_int32), _p(val, C.c_double), _p(mass, C.c_double), float(g))
    else:
        args = (None, None, None, None, 0.0)
    ptr = L.orc_run(_p(v, C.c_double), len(v), _p(f, C.c_uint32), len(f), *args, seed, _p(cfg, C.c_double))
    try:
        out = json.loads(C.string_at(ptr).decode())
    finally:
        L.orc_free(ptr)
    del keep
    out["hashes"] = [int(h) for h in out.get("hashes", [])]
    return out
