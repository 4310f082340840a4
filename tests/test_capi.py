"""The C-ABI library: loads, exports every symbol include/difftopo_b200.h
declares, and fails loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import pytest

import paper_2105_13168_b200 as dt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "difftopo_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dtb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(dt.LIB_PATH)
    names = declared()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    dt.load_library()
    import inspect
    src = inspect.getsource(dt.load_library)
    missing = [n for n in declared() if f'"{n}"' not in src]
    assert not missing, missing


def test_config_defaults_match_reference():
    c = dt.default_config()
    assert (c.band_low_threshold, c.saturation, c.collision_threshold, c.check_interval, c.max_steps,
            c.covered_threshold, c.record_trails) == (0.05, 0.999, 0.1, 1, 200000, 0.05, 1)
    k = dt.default_coefficients()
    assert (k.gradient_energy, k.penalty, k.contact, k.mobility) == (1 / 25, 1 / 125, 1 / 30, 0.25)


def _has_gpu():
    try:
        return dt.device_info()["devices"] > 0
    except dt.DiffTopoError:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_device_calls_fail_loudly_without_gpu():
    m = dt.TriangleMesh.generate("torus:16:8:2:0.5")  # host-only: fine
    with pytest.raises(dt.DiffTopoError) as e:
        dt.assemble_laplacian(m)
    assert e.value.kind == "CudaError"
    with pytest.raises(dt.DiffTopoError):
        dt.LayerField(m, [0])


def test_cpp_facade_compiles(tmp_path):
    """The C++ drop-in header (include/difftopo_b200.hpp) compiles and links
    against the library exactly as a reference user's program would."""
    import subprocess
    exe = tmp_path / "detect_loops"
    subprocess.run(["g++", "-O2", "-std=c++17", "-Wall", "-Werror", f"-I{ROOT}/include",
                    f"{ROOT}/examples/detect_loops.cpp", f"-L{ROOT}/paper_2105_13168_b200/lib", "-ldifftopo_b200",
                    f"-Wl,-rpath,{ROOT}/paper_2105_13168_b200/lib", "-o", str(exe)], check=True)
    assert exe.exists()


_CONN_PROBE = (
    "import ctypes, sys; sys.path.insert(0, {root!r}); import paper_2105_13168_b200 as dt; dt.load_library(); "
    "{init}"
    "libc = ctypes.CDLL(None); libc.getenv.restype = ctypes.c_char_p; "
    "print((libc.getenv(b'CUDA_DEVICE_MAX_CONNECTIONS') or b'-').decode())"
)


@pytest.mark.parametrize("preset,init,expect", [(None, False, "-"), (None, True, "32"), ("4", True, "4")])
def test_work_queues_are_opt_in(preset, init, expect):
    """Loading the library leaves CUDA_DEVICE_MAX_CONNECTIONS alone;
    dtb_init_work_queues (before any CUDA context) sets it when the caller
    left it unset, and a value the caller set is kept."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    if preset is not None:
        env["CUDA_DEVICE_MAX_CONNECTIONS"] = preset
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _CONN_PROBE.format(root=root, init="dt.init_work_queues(32); " if init else "")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True,
                         timeout=120)
    assert out.stdout.strip() == expect


def test_work_queues_rejects_bad_count():
    import paper_2105_13168_b200 as dt
    with pytest.raises(dt.DiffTopoError):
        dt.init_work_queues(0)
