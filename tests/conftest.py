import ctypes
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HELPERS = os.path.join(ROOT, "tests", "helpers")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); runs through the C-ABI library")
    config.addinivalue_line("markers", "slow: long CPU test (still part of the default suite unless deselected)")


def _build(src, out, cmd):
    if not os.path.exists(out) or os.path.getmtime(src) > os.path.getmtime(out):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(cmd + ["-o", tmp, src])
        os.replace(tmp, out)
    return out


@pytest.fixture(scope="session")
def curand_ref():
    """cuRAND's Philox4x32-10, host-compiled (library routine used as a pin)."""
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the cuRAND host helper")
    src = os.path.join(HELPERS, "curand_philox_host.cu")
    out = os.path.join(HELPERS, "libcurand_philox_host.so")
    _build(src, out, [nvcc, "-O2", "-shared", "-Xcompiler", "-fPIC", "-x", "cu"])
    lib = ctypes.CDLL(out)
    lib.curand_ref_philox.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64]
    return lib


@pytest.fixture(scope="session")
def lemire_enum():
    src = os.path.join(HELPERS, "lemire_enum.c")
    out = os.path.join(HELPERS, "liblemire_enum.so")
    _build(src, out, ["gcc", "-O2", "-shared", "-fPIC"])
    lib = ctypes.CDLL(out)
    lib.lemire32_enumerate.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
    lib.lemire16_enumerate.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
    return lib
