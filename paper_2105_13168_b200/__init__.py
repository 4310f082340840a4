"""Python view of the B200 diffusion-front engine (ctypes over the C ABI).

The product is ``lib/libdifftopo_b200.so`` (include/difftopo_b200.h); this
module mirrors the reference's C++ API names (proj/include/difftopo/*.hpp:
``TriangleMesh``, ``assemble_laplacian``, ``run_initial_pass``,
``extract_front``, ``detect_collisions``, ``build_reeb`` ...) for tests and
benchmarks.  There is no CPU fallback: importing works without a GPU, but any
device call raises ``DiffTopoError`` (code DTB_ECUDA) when no sm_100a device is
present, and a missing shared library raises ``ImportError`` at load.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTB_LIBRARY") or os.path.join(_HERE, "lib", "libdifftopo_b200.so")  # override: A/B runs

ERRORS = {
    1: "ParseError", 2: "TopologyError", 3: "DegeneracyError", 4: "InvalidParameter",
    5: "DimensionMismatch", 6: "EmptySeed", 7: "ZeroColumn", 8: "InvalidSplit", 9: "InvalidMerge",
    10: "NumericalBlowup", 11: "MaxStepsExceeded", 12: "Unreachable", 13: "StallError",
    14: "LoopError", 15: "InconsistentLog", 100: "CudaError", 101: "CapacityExceeded",
}
EVENT_KINDS = ("seed", "split", "merge", "vanish")


class DiffTopoError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"{ERRORS.get(code, code)}: {message}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class Config(C.Structure):
    """DiffusionConfig (diffusion.hpp:33)."""

    _fields_ = [
        ("dt", C.c_double), ("band_low_threshold", C.c_double), ("saturation", C.c_double),
        ("collision_threshold", C.c_double), ("check_interval", C.c_int32), ("record_trails", C.c_int32),
        ("max_steps", C.c_int64), ("covered_threshold", C.c_double), ("seed_radius", C.c_double),
        ("record_hashes", C.c_int32), ("grid_ctas", C.c_int32),
    ]


class Coefficients(C.Structure):
    """CoefficientScheme (layer_field.hpp:30)."""

    _fields_ = [("gradient_energy", C.c_double), ("penalty", C.c_double), ("contact", C.c_double),
                ("mobility", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    P, U32, I32, I64, D = C.c_void_p, C.c_uint32, C.c_int32, C.c_int64, C.c_double
    pU32, pI32, pI64, pD, pU64 = (C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_double), C.POINTER(C.c_uint64))
    pP = C.POINTER(C.c_void_p)
    sig = {
        "dtb_config_default": (None, [C.POINTER(Config)]),
        "dtb_coefficients_default": (None, [C.POINTER(Coefficients)]),
        "dtb_last_error": (C.c_char_p, []),
        "dtb_version": (C.c_char_p, []),
        "dtb_warmup": (C.c_int, []),
        "dtb_init_work_queues": (C.c_int, [I32]),
        "dtb_device_info": (C.c_int, [pI32, pI32, pI32, pI32]),
        "dtb_mesh_from_arrays": (C.c_int, [pD, U32, pU32, U32, pP]),
        "dtb_mesh_generate": (C.c_int, [C.c_char_p, pP]),
        "dtb_mesh_load": (C.c_int, [C.c_char_p, I32, pP]),
        "dtb_mesh_save": (C.c_int, [P, C.c_char_p]),
        "dtb_mesh_free": (None, [P]),
        "dtb_mesh_info": (C.c_int, [P, pU32, pU32, pU32, pI64, pI64]),
        "dtb_mesh_vertices": (C.c_int, [P, pD]),
        "dtb_mesh_faces": (C.c_int, [P, pU32]),
        "dtb_mesh_edges": (C.c_int, [P, pU32, pU32]),
        "dtb_mesh_face_edges": (C.c_int, [P, pU32]),
        "dtb_mesh_adjacency": (C.c_int, [P, pU32, pU32, pU32, pU32]),
        "dtb_seed_region": (C.c_int, [P, U32, D, pU32, U32, pU32]),
        "dtb_laplacian_assemble": (C.c_int, [P, pP]),
        "dtb_laplacian_from_csr": (C.c_int, [P, pI32, pI32, pD, pD, I64, D, pP]),
        "dtb_laplacian_free": (None, [P]),
        "dtb_laplacian_info": (C.c_int, [P, pI64, pD]),
        "dtb_laplacian_csr": (C.c_int, [P, pI32, pI32, pD, pD]),
        "dtb_laplacian_apply": (C.c_int, [P, pD, pD]),
        "dtb_laplacian_sweep_bench": (C.c_int, [P, C.c_int32, pD, pD]),
        "dtb_stable_time_step": (C.c_int, [P, C.POINTER(Coefficients), pD]),
        "dtb_run_initial_pass": (C.c_int, [P, P, U32, C.POINTER(Config), C.POINTER(Coefficients), pP]),
        "dtb_run_initial_pass_batch": (C.c_int, [pP, pP, pU32, C.c_int32, C.POINTER(Config),
                                                 C.POINTER(Coefficients), C.c_int32, pP, pI32]),
        "dtb_result_free": (None, [P]),
        "dtb_result_summary": (C.c_int, [P, pI32, pI64, pD, pI64, pI64, pI64, pI64]),
        "dtb_result_message": (C.c_char_p, [P]),
        "dtb_result_event": (C.c_int, [P, I64, pI32, pI64, pD, pU32, pU32, pU32, pU32]),
        "dtb_result_event_layers": (C.c_int, [P, I64, pU32, pU32]),
        "dtb_result_event_covered": (C.c_int, [P, I64, pU32]),
        "dtb_result_estimate": (C.c_int, [P, I64, U32, pU32, pU32, pU32, pD]),
        "dtb_result_estimate_points": (C.c_int, [P, I64, U32, pI64, pD, pI64, pD]),
        "dtb_result_estimate_snapshot": (C.c_int, [P, I64, U32, pU32, pD]),
        "dtb_result_track": (C.c_int, [P, I64, pI64, pI64, pI64, pU32]),
        "dtb_result_track_trail": (C.c_int, [P, I64, pD]),
        "dtb_result_layer": (C.c_int, [P, U32, pI32, pI32, pI64, pI64, pU32]),
        "dtb_result_layer_values": (C.c_int, [P, U32, pU32, pD, U32, pU32]),
        "dtb_result_field_hash": (C.c_int, [P, pU64]),
        "dtb_result_hashes": (C.c_int, [P, pU64, I64, pI64]),
        "dtb_result_timing": (C.c_int, [P, pD, pD, pI64, pI64, pI64]),
        "dtb_result_reeb": (C.c_int, [P, pI64, pI64, pI64]),
        "dtb_result_work": (C.c_int, [P, pU64, pU64, pD, pD]),
        "dtb_launch_count": (C.c_ulonglong, []),
        "dtb_bench_barrier": (C.c_double, [C.c_int, C.c_int, C.c_int]),
        "dtb_mesh_device_bytes": (C.c_int, [P, pU64]),
        "dtb_mesh_upload_bytes": (C.c_int, [P, pU64]),
        "dtb_result_reeb_arcs": (C.c_int, [P, pU32, pU32, pU32]),
        "dtb_field_init": (C.c_int, [P, pU32, U32, pP]),
        "dtb_field_free": (None, [P]),
        "dtb_field_step": (C.c_int, [P, P, C.POINTER(Config), C.POINTER(Coefficients)]),
        "dtb_field_layer_count": (C.c_int, [P, pU32]),
        "dtb_field_layer_values": (C.c_int, [P, U32, pU32, pD, U32, pU32]),
        "dtb_field_hash": (C.c_int, [P, pU64]),
        "dtb_field_normalize": (C.c_int, [P]),
        "dtb_field_covered_set": (C.c_int, [P, D, pU32, U32, pU32]),
        "dtb_field_extract_front": (C.c_int, [P, U32, C.POINTER(Config), pU32, pU32, pU32, pD, pU32, pU32]),
        "dtb_field_detect_collisions": (C.c_int, [P, C.POINTER(Config), pU32, pU32, U32, pU32, pU32]),
        "dtb_field_split_layer": (C.c_int, [P, U32, pU32, pU32, U32, I64, pU32]),
        "dtb_field_merge_layers": (C.c_int, [P, pU32, U32, I64, pU32]),
        "dtb_extract_isoline": (C.c_int, [P, pD, D, pU32, pU32, pI64, pD, pI64, pD, U32]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("DTB_LIBRARY") and not hasattr(lib, name):
            continue  # an older build under A/B comparison
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = None  # filled lazily for tests


def _check(rc: int):
    if rc != 0:
        raise DiffTopoError(rc, _lib.dtb_last_error().decode())


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def default_config(**overrides) -> Config:
    lib = load_library()
    c = Config()
    lib.dtb_config_default(C.byref(c))
    for k, v in overrides.items():
        if not hasattr(c, k):
            raise AttributeError(k)
        setattr(c, k, v)
    return c


def default_coefficients(**overrides) -> Coefficients:
    lib = load_library()
    c = Coefficients()
    lib.dtb_coefficients_default(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def launch_count() -> int:
    return int(load_library().dtb_launch_count())


def device_info():
    lib = load_library()
    n, sms, ma, mi = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib.dtb_device_info(C.byref(n), C.byref(sms), C.byref(ma), C.byref(mi))
    _check(rc)
    return {"devices": n.value, "sms": sms.value, "cc": (ma.value, mi.value)}


def init_work_queues(queues: int = 32):
    """Opt-in: request `queues` hardware work queues for the CUDA context this
    process is about to create (dtb_init_work_queues; concurrent batch passes
    hold one each).  Must run before any CUDA use; raises if a context may
    already exist."""
    _check(load_library().dtb_init_work_queues(int(queues)))


def warmup():
    """Creates the CUDA context and loads the library's kernels with one small
    end-to-end call (dtb_warmup), so the first real call is not a cold one."""
    _check(load_library().dtb_warmup())


class TriangleMesh:
    """TriangleMesh (mesh.hpp:33): validated, oriented, indexed on the host;
    copied to HBM on first device use."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_arrays(cls, vertices, faces) -> "TriangleMesh":
        lib = load_library()
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        f = np.ascontiguousarray(faces, dtype=np.uint32).reshape(-1, 3)
        h = C.c_void_p()
        _check(lib.dtb_mesh_from_arrays(_ptr(v, C.c_double), v.shape[0], _ptr(f, C.c_uint32), f.shape[0],
                                        C.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, spec: str) -> "TriangleMesh":
        lib = load_library()
        h = C.c_void_p()
        _check(lib.dtb_mesh_generate(spec.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str, fmt: int = 0) -> "TriangleMesh":
        lib = load_library()
        h = C.c_void_p()
        _check(lib.dtb_mesh_load(path.encode(), fmt, C.byref(h)))
        return cls(h)

    def device_bytes(self) -> int:
        b = C.c_uint64()
        _check(_lib.dtb_mesh_device_bytes(self._h, C.byref(b)))
        return b.value

    def upload_bytes(self) -> int:
        """Host->device bytes of this mesh's device copy (builds it if needed)."""
        b = C.c_uint64()
        _check(_lib.dtb_mesh_upload_bytes(self._h, C.byref(b)))
        return b.value

    def save(self, path: str):
        _check(_lib.dtb_mesh_save(self._h, path.encode()))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dtb_mesh_free(self._h)
            self._h = None

    def info(self):
        nv, ne, nf, eu, g = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_int64(), C.c_int64()
        _check(_lib.dtb_mesh_info(self._h, C.byref(nv), C.byref(ne), C.byref(nf), C.byref(eu), C.byref(g)))
        return {"V": nv.value, "E": ne.value, "F": nf.value, "euler": eu.value, "genus": g.value}

    @property
    def vertex_count(self):
        return self.info()["V"]

    def vertices(self) -> np.ndarray:
        out = np.empty((self.info()["V"], 3), np.float64)
        _check(_lib.dtb_mesh_vertices(self._h, _ptr(out, C.c_double)))
        return out

    def faces(self) -> np.ndarray:
        out = np.empty((self.info()["F"], 3), np.uint32)
        _check(_lib.dtb_mesh_faces(self._h, _ptr(out, C.c_uint32)))
        return out

    def edges(self) -> Tuple[np.ndarray, np.ndarray]:
        ne = self.info()["E"]
        ev = np.empty((ne, 2), np.uint32)
        ef = np.empty((ne, 2), np.uint32)
        _check(_lib.dtb_mesh_edges(self._h, _ptr(ev, C.c_uint32), _ptr(ef, C.c_uint32)))
        return ev, ef

    def face_edges(self) -> np.ndarray:
        out = np.empty((self.info()["F"], 3), np.uint32)
        _check(_lib.dtb_mesh_face_edges(self._h, _ptr(out, C.c_uint32)))
        return out

    def adjacency(self):
        """(v2v_off, v2v, v2f_off, v2f): sorted vertex neighbours and incident
        faces in face order (mesh.hpp:57-62)."""
        i = self.info()
        vo, vv = np.empty(i["V"] + 1, np.uint32), np.empty(2 * i["E"], np.uint32)
        fo, ff = np.empty(i["V"] + 1, np.uint32), np.empty(3 * i["F"], np.uint32)
        _check(_lib.dtb_mesh_adjacency(self._h, _ptr(vo, C.c_uint32), _ptr(vv, C.c_uint32), _ptr(fo, C.c_uint32),
                                       _ptr(ff, C.c_uint32)))
        return vo, vv, fo, ff

    def seed_region(self, seed: int, radius: float) -> np.ndarray:
        n = C.c_uint32()
        _check(_lib.dtb_seed_region(self._h, seed, radius, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        _check(_lib.dtb_seed_region(self._h, seed, radius, _ptr(out, C.c_uint32), n.value, C.byref(n)))
        return out


def topology_summary(mesh: TriangleMesh):
    return mesh.info()


class LaplacianOperator:
    """LaplacianOperator (operators.hpp:16), resident in HBM."""

    def __init__(self, handle, mesh):
        self._h = handle
        self.mesh = mesh

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dtb_laplacian_free(self._h)
            self._h = None

    @classmethod
    def from_csr(cls, mesh: TriangleMesh, off, col, val, mass, gershgorin: float) -> "LaplacianOperator":
        off = np.ascontiguousarray(off, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        mass = np.ascontiguousarray(mass, np.float64)
        h = C.c_void_p()
        _check(load_library().dtb_laplacian_from_csr(mesh._h, _ptr(off, C.c_int32), _ptr(col, C.c_int32),
                                                     _ptr(val, C.c_double), _ptr(mass, C.c_double), len(col),
                                                     float(gershgorin), C.byref(h)))
        return cls(h, mesh)

    def info(self):
        nnz, g = C.c_int64(), C.c_double()
        _check(_lib.dtb_laplacian_info(self._h, C.byref(nnz), C.byref(g)))
        return nnz.value, g.value

    @property
    def gershgorin_bound(self):
        return self.info()[1]

    def csr(self):
        nnz, _ = self.info()
        nv = self.mesh.vertex_count
        off = np.empty(nv + 1, np.int32)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        mass = np.empty(nv, np.float64)
        _check(_lib.dtb_laplacian_csr(self._h, _ptr(off, C.c_int32), _ptr(col, C.c_int32), _ptr(val, C.c_double),
                                      _ptr(mass, C.c_double)))
        return off, col, val, mass

    def apply(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        _check(_lib.dtb_laplacian_apply(self._h, _ptr(x, C.c_double), _ptr(y, C.c_double)))
        return y

    def sweep_bench(self, reps: int = 10) -> dict:
        """Diagnostics: one full-mesh sweep of the operator (the padded-row
        SpMV ``apply`` runs) timed on the device after an L2 flush; mean
        seconds and algorithmic bytes per sweep."""
        sec, nbytes = C.c_double(), C.c_double()
        _check(_lib.dtb_laplacian_sweep_bench(self._h, int(reps), C.byref(sec), C.byref(nbytes)))
        return {"seconds": sec.value, "bytes": nbytes.value, "gbs": nbytes.value / sec.value / 1e9}


def assemble_laplacian(mesh: TriangleMesh) -> LaplacianOperator:
    h = C.c_void_p()
    _check(load_library().dtb_laplacian_assemble(mesh._h, C.byref(h)))
    return LaplacianOperator(h, mesh)


def stable_time_step(op: LaplacianOperator, coefficients: Optional[Coefficients] = None) -> float:
    dt = C.c_double()
    co = coefficients or default_coefficients()
    _check(_lib.dtb_stable_time_step(op._h, C.byref(co), C.byref(dt)))
    return dt.value


@dataclass
class LoopPoint:
    edge: int
    t: float
    face: int
    position: Tuple[float, float, float]


@dataclass
class HandleEstimate:
    layer: int
    length: float
    points: List[LoopPoint]
    snapshot: Tuple[np.ndarray, np.ndarray]


@dataclass
class TopologyEvent:
    kind: str
    step: int
    layers: List[int]
    produced: List[int]
    position: Tuple[float, float, float]
    estimates: List[HandleEstimate] = field(default_factory=list)
    covered: Optional[np.ndarray] = None


class InitialPassResult:
    """InitialPassResult (diffusion.hpp:110).  Unlike the reference, a run that
    ends in an error keeps its partial event log; ``status`` names the error."""

    def __init__(self, handle):
        self._h = handle
        st, steps, dt, ne, nt, nest, lc = (C.c_int32(), C.c_int64(), C.c_double(), C.c_int64(), C.c_int64(),
                                           C.c_int64(), C.c_int64())
        _check(_lib.dtb_result_summary(self._h, C.byref(st), C.byref(steps), C.byref(dt), C.byref(ne), C.byref(nt),
                                       C.byref(nest), C.byref(lc)))
        self.status_code = st.value
        self.status = "ok" if st.value == 0 else ERRORS.get(st.value, str(st.value))
        self.message = _lib.dtb_result_message(self._h).decode()
        self.steps = steps.value
        self.dt_used = dt.value
        self.n_events = ne.value
        self.n_tracks = nt.value
        self.handle_estimate_count = nest.value
        self.layer_count = lc.value
        self._events = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dtb_result_free(self._h)
            self._h = None

    def events(self, with_covered: bool = True) -> List[TopologyEvent]:
        if self._events is not None:
            return self._events
        out = []
        for i in range(self.n_events):
            kind, step = C.c_int32(), C.c_int64()
            pos = np.empty(3, np.float64)
            nl, np_, ne, nc = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
            _check(_lib.dtb_result_event(self._h, i, C.byref(kind), C.byref(step), _ptr(pos, C.c_double),
                                         C.byref(nl), C.byref(np_), C.byref(ne), C.byref(nc)))
            layers = np.empty(max(1, nl.value), np.uint32)
            prod = np.empty(max(1, np_.value), np.uint32)
            _check(_lib.dtb_result_event_layers(self._h, i, _ptr(layers, C.c_uint32), _ptr(prod, C.c_uint32)))
            cov = None
            if with_covered:
                cov = np.empty(max(1, nc.value), np.uint32)
                _check(_lib.dtb_result_event_covered(self._h, i, _ptr(cov, C.c_uint32)))
                cov = cov[: nc.value]
            ests = []
            for k in range(ne.value):
                lay, npts, nsnap, length = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_double()
                _check(_lib.dtb_result_estimate(self._h, i, k, C.byref(lay), C.byref(npts), C.byref(nsnap),
                                                C.byref(length)))
                e = np.empty(npts.value, np.int64)
                t = np.empty(npts.value, np.float64)
                f = np.empty(npts.value, np.int64)
                xyz = np.empty((npts.value, 3), np.float64)
                _check(_lib.dtb_result_estimate_points(self._h, i, k, _ptr(e, C.c_int64), _ptr(t, C.c_double),
                                                       _ptr(f, C.c_int64), _ptr(xyz, C.c_double)))
                sv = np.empty(nsnap.value, np.uint32)
                sx = np.empty(nsnap.value, np.float64)
                _check(_lib.dtb_result_estimate_snapshot(self._h, i, k, _ptr(sv, C.c_uint32), _ptr(sx, C.c_double)))
                pts = [LoopPoint(int(e[j]), float(t[j]), int(f[j]), tuple(xyz[j])) for j in range(npts.value)]
                ests.append(HandleEstimate(lay.value, length.value, pts, (sv, sx)))
            out.append(TopologyEvent(EVENT_KINDS[kind.value], step.value, [int(x) for x in layers[: nl.value]],
                                     [int(x) for x in prod[: np_.value]], tuple(pos), ests, cov))
        self._events = out
        return out

    def tracks(self):
        out = []
        for i in range(self.n_tracks):
            layer, cr, co, nt = C.c_int64(), C.c_int64(), C.c_int64(), C.c_uint32()
            _check(_lib.dtb_result_track(self._h, i, C.byref(layer), C.byref(cr), C.byref(co), C.byref(nt)))
            trail = np.empty((nt.value, 3), np.float64)
            if nt.value:
                _check(_lib.dtb_result_track_trail(self._h, i, _ptr(trail, C.c_double)))
            out.append({"layer": layer.value, "created": cr.value, "consumed": co.value, "trail": trail})
        return out

    def layer_table(self):
        out = []
        for lid in range(self.layer_count):
            a, c, p, cs, nmp = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_uint32()
            _check(_lib.dtb_result_layer(self._h, lid, C.byref(a), C.byref(c), C.byref(p), C.byref(cs),
                                         C.byref(nmp)))
            out.append({"id": lid, "active": a.value, "cleared": c.value, "parent": p.value,
                        "created_step": cs.value})
        return out

    def layer_values(self, layer: int):
        n = C.c_uint32()
        _check(_lib.dtb_result_layer_values(self._h, layer, None, None, 0, C.byref(n)))
        v = np.empty(n.value, np.uint32)
        x = np.empty(n.value, np.float64)
        _check(_lib.dtb_result_layer_values(self._h, layer, _ptr(v, C.c_uint32), _ptr(x, C.c_double), n.value,
                                            C.byref(n)))
        return v, x

    def field_hash(self) -> int:
        h = C.c_uint64()
        _check(_lib.dtb_result_field_hash(self._h, C.byref(h)))
        return h.value

    def hashes(self) -> np.ndarray:
        n = C.c_int64()
        _check(_lib.dtb_result_hashes(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint64)
        _check(_lib.dtb_result_hashes(self._h, _ptr(out, C.c_uint64), n.value, C.byref(n)))
        return out

    def timing(self):
        td, te, la, ec, ks = C.c_double(), C.c_double(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.dtb_result_timing(self._h, C.byref(td), C.byref(te), C.byref(la), C.byref(ec), C.byref(ks)))
        sr, si, tp, tk = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_double()
        _check(_lib.dtb_result_work(self._h, C.byref(sr), C.byref(si), C.byref(tp), C.byref(tk)))
        return {"t_device": td.value, "t_events": te.value, "launches": la.value, "event_checks": ec.value,
                "kernel_steps": ks.value, "sum_region": sr.value, "sum_interest": si.value,
                "t_pass_device": tp.value, "t_kernel": tk.value}

    def reeb(self):
        nn, na, rank = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.dtb_result_reeb(self._h, C.byref(nn), C.byref(na), C.byref(rank)))
        fr = np.empty(max(1, na.value), np.uint32)
        to = np.empty(max(1, na.value), np.uint32)
        ly = np.empty(max(1, na.value), np.uint32)
        _check(_lib.dtb_result_reeb_arcs(self._h, _ptr(fr, C.c_uint32), _ptr(to, C.c_uint32), _ptr(ly, C.c_uint32)))
        arcs = [(int(fr[i]), int(to[i]), int(ly[i])) for i in range(na.value)]
        return {"nodes": nn.value, "arcs": arcs, "cycle_rank": rank.value}


def run_initial_pass(mesh: TriangleMesh, op: LaplacianOperator, seed_vertex: int = 0,
                     cfg: Optional[Config] = None, coefficients: Optional[Coefficients] = None) -> InitialPassResult:
    lib = load_library()
    cfg = cfg or default_config()
    co = coefficients or default_coefficients()
    h = C.c_void_p()
    _check(lib.dtb_run_initial_pass(mesh._h, op._h, seed_vertex, C.byref(cfg), C.byref(co), C.byref(h)))
    return InitialPassResult(h)


def run_initial_pass_batch(meshes: Sequence[TriangleMesh], ops: Sequence[LaplacianOperator],
                           seeds: Optional[Sequence[int]] = None, cfg: Optional[Config] = None,
                           coefficients: Optional[Coefficients] = None,
                           concurrency: int = 0) -> List[InitialPassResult]:
    """Independent initial passes of a batch of meshes on this GPU, several at
    once (dtb_run_initial_pass_batch); item i equals
    run_initial_pass(meshes[i], ops[i], seeds[i], cfg)."""
    lib = load_library()
    n = len(meshes)
    if len(ops) != n or (seeds is not None and len(seeds) != n):
        raise ValueError("meshes, ops and seeds must have the same length")
    cfg = cfg or default_config()
    co = coefficients or default_coefficients()
    mh = (C.c_void_p * max(1, n))(*[m._h for m in meshes])
    oh = (C.c_void_p * max(1, n))(*[o._h for o in ops])
    sd = np.ascontiguousarray(seeds if seeds is not None else np.zeros(n), np.uint32)
    out = (C.c_void_p * max(1, n))()
    rc = np.zeros(max(1, n), np.int32)
    code = lib.dtb_run_initial_pass_batch(mh, oh, _ptr(sd, C.c_uint32), n, C.byref(cfg), C.byref(co), concurrency,
                                          out, _ptr(rc, C.c_int32))
    err = DiffTopoError(code, lib.dtb_last_error().decode()) if code else None  # before other calls reset it
    results = [InitialPassResult(C.c_void_p(out[i])) if out[i] else None for i in range(n)]
    if err is not None:
        raise err
    return results


class LayerField:
    """LayerField (layer_field.hpp:46) with the one-shot operations."""

    def __init__(self, mesh: TriangleMesh, seeds: Sequence[int]):
        s = np.ascontiguousarray(seeds, np.uint32)
        h = C.c_void_p()
        _check(load_library().dtb_field_init(mesh._h, _ptr(s, C.c_uint32), len(s), C.byref(h)))
        self._h = h
        self.mesh = mesh

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.dtb_field_free(self._h)
            self._h = None

    @property
    def layer_count(self) -> int:
        n = C.c_uint32()
        _check(_lib.dtb_field_layer_count(self._h, C.byref(n)))
        return n.value

    def step(self, op: LaplacianOperator, cfg: Optional[Config] = None, coefficients=None):
        cfg = cfg or default_config()
        co = coefficients or default_coefficients()
        _check(_lib.dtb_field_step(self._h, op._h, C.byref(cfg), C.byref(co)))

    def layer_values(self, layer: int):
        n = C.c_uint32()
        _check(_lib.dtb_field_layer_values(self._h, layer, None, None, 0, C.byref(n)))
        v = np.empty(n.value, np.uint32)
        x = np.empty(n.value, np.float64)
        _check(_lib.dtb_field_layer_values(self._h, layer, _ptr(v, C.c_uint32), _ptr(x, C.c_double), n.value,
                                           C.byref(n)))
        return v, x

    def hash(self) -> int:
        h = C.c_uint64()
        _check(_lib.dtb_field_hash(self._h, C.byref(h)))
        return h.value

    def normalize_columns(self):
        _check(_lib.dtb_field_normalize(self._h))

    def covered_set(self, threshold: float) -> np.ndarray:
        n = C.c_uint32()
        _check(_lib.dtb_field_covered_set(self._h, threshold, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        _check(_lib.dtb_field_covered_set(self._h, threshold, _ptr(out, C.c_uint32), n.value, C.byref(n)))
        return out

    def extract_front(self, layer: int, cfg: Optional[Config] = None):
        cfg = cfg or default_config()
        n = C.c_uint32()
        _check(_lib.dtb_field_extract_front(self._h, layer, C.byref(cfg), C.byref(n), None, None, None, None, None))
        tc = np.empty(max(1, n.value), np.uint32)
        bc = np.empty(max(1, n.value), np.uint32)
        bl = np.empty(max(1, n.value), np.float64)
        _check(_lib.dtb_field_extract_front(self._h, layer, C.byref(cfg), C.byref(n), _ptr(tc, C.c_uint32),
                                            _ptr(bc, C.c_uint32), _ptr(bl, C.c_double), None, None))
        tris = np.empty(max(1, int(tc[: n.value].sum())), np.uint32)
        bnd = np.empty(max(1, int(bc[: n.value].sum())), np.uint32)
        _check(_lib.dtb_field_extract_front(self._h, layer, C.byref(cfg), C.byref(n), None, None, None,
                                            _ptr(tris, C.c_uint32), _ptr(bnd, C.c_uint32)))
        comps, ot, ob = [], 0, 0
        for i in range(n.value):
            comps.append({"triangles": tris[ot: ot + tc[i]].tolist(), "boundary": bnd[ob: ob + bc[i]].tolist(),
                          "band_length": float(bl[i])})
            ot += int(tc[i])
            ob += int(bc[i])
        return comps

    def detect_collisions(self, cfg: Optional[Config] = None):
        cfg = cfg or default_config()
        ng, nf = C.c_uint32(), C.c_uint32()
        _check(_lib.dtb_field_detect_collisions(self._h, C.byref(cfg), None, None, 0, C.byref(ng), C.byref(nf)))
        flat = np.empty(max(1, nf.value), np.uint32)
        sizes = np.empty(max(1, ng.value), np.uint32)
        _check(_lib.dtb_field_detect_collisions(self._h, C.byref(cfg), _ptr(flat, C.c_uint32),
                                                _ptr(sizes, C.c_uint32), nf.value, C.byref(ng), C.byref(nf)))
        out, o = [], 0
        for i in range(ng.value):
            out.append(flat[o: o + sizes[i]].tolist())
            o += int(sizes[i])
        return out

    def split_layer(self, layer: int, components: Sequence[Sequence[int]], step: int = 0) -> List[int]:
        flat = np.ascontiguousarray(np.concatenate([np.asarray(c, np.uint32) for c in components]), np.uint32)
        sizes = np.asarray([len(c) for c in components], np.uint32)
        ch = np.empty(len(components), np.uint32)
        _check(_lib.dtb_field_split_layer(self._h, layer, _ptr(flat, C.c_uint32), _ptr(sizes, C.c_uint32),
                                          len(components), step, _ptr(ch, C.c_uint32)))
        return ch.tolist()

    def merge_layers(self, ids: Sequence[int], step: int = 0) -> int:
        a = np.ascontiguousarray(ids, np.uint32)
        r = C.c_uint32()
        _check(_lib.dtb_field_merge_layers(self._h, _ptr(a, C.c_uint32), len(a), step, C.byref(r)))
        return r.value


def extract_isoline(mesh: TriangleMesh, values, level: float):
    vals = np.ascontiguousarray(values, np.float64)
    n = C.c_uint32()
    lib = load_library()
    _check(lib.dtb_extract_isoline(mesh._h, _ptr(vals, C.c_double), level, C.byref(n), None, None, None, None, None,
                                   0))
    counts = np.empty(max(1, n.value), np.uint32)
    _check(lib.dtb_extract_isoline(mesh._h, _ptr(vals, C.c_double), level, C.byref(n), _ptr(counts, C.c_uint32),
                                   None, None, None, None, 0))
    total = int(counts[: n.value].sum())
    e = np.empty(max(1, total), np.int64)
    t = np.empty(max(1, total), np.float64)
    f = np.empty(max(1, total), np.int64)
    xyz = np.empty((max(1, total), 3), np.float64)
    _check(lib.dtb_extract_isoline(mesh._h, _ptr(vals, C.c_double), level, C.byref(n), _ptr(counts, C.c_uint32),
                                   _ptr(e, C.c_int64), _ptr(t, C.c_double), _ptr(f, C.c_int64),
                                   _ptr(xyz, C.c_double), total))
    loops, o = [], 0
    for i in range(n.value):
        c = int(counts[i])
        loops.append([LoopPoint(int(e[o + j]), float(t[o + j]), int(f[o + j]), tuple(xyz[o + j])) for j in range(c)])
        o += c
    return loops
