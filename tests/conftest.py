import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def golden(name="examples.json"):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


_PIN_SRC = os.path.join(ROOT, "tests", "pins", "curand_pin.cu")
_PIN_LIB = os.path.join(ROOT, "tests", "pins", "libcurandpin.so")


@pytest.fixture(scope="session")
def curand_pin():
    """Host-compiled cuRAND Philox4_32_10 device-API code (a library routine)."""
    import ctypes
    if not os.path.exists(_PIN_LIB) or os.path.getmtime(_PIN_LIB) < os.path.getmtime(_PIN_SRC):
        tmp = _PIN_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-Xcompiler", "-fPIC", "-shared", "-O2",
                               "-Wno-deprecated-gpu-targets", "-o", tmp, _PIN_SRC])
        os.replace(tmp, _PIN_LIB)
    lib = ctypes.CDLL(_PIN_LIB)
    P = ctypes.c_void_p
    u64, i64 = ctypes.c_uint64, ctypes.c_int64
    lib.pin_curand4.argtypes = [u64, u64, u64, i64, P]
    lib.pin_philox_block.argtypes = [P, P, P]
    lib.pin_curand_normal4.argtypes = [u64, u64, u64, i64, P]
    return lib


def np_ptr(a):
    import ctypes
    return ctypes.c_void_p(a.ctypes.data)


def row_rel_err(a, b):
    """max_i max_c |a_ic - b_ic| / ||b_i||_2 (the north-star parity metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nrm = np.linalg.norm(b, axis=1, keepdims=True)
    nrm = np.where(nrm > 0, nrm, 1.0)
    return float(np.max(np.abs(a - b) / nrm)) if a.size else 0.0


_RECORDS = {}


def record(name, value):
    """Collect parity numbers; written to $IGP_PARITY_LOG at session end (if set)."""
    _RECORDS[name] = value


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("IGP_PARITY_LOG")
    if path and _RECORDS:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(_RECORDS, f, indent=1, sort_keys=True)
