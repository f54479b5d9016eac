"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/shuf.h declares, and validates arguments without a GPU
(no compute calls here)."""
import ctypes
import os
import re

import pytest

import paper_2302_03317_b200 as shuf
from paper_2302_03317_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    _build.build()
    return shuf.lib()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "shuf.h")).read()
    return sorted(set(re.findall(r"\b(shuf_[a-z_]+)\s*\(", hdr)))


def test_header_declares_what_binding_exports():
    assert declared_symbols() == sorted(shuf.EXPORTED_SYMBOLS)


def test_every_declared_symbol_is_exported(L):
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_sm100a_code_in_library():
    out = os.popen(f"cuobjdump -lelf {shuf.lib_path} 2>&1").read()
    assert "sm_100a" in out, out


@pytest.mark.parametrize("args,code", [
    ((100, 257, 256, 16, 1), 2),    # elem_bytes above 256: unsupported on device
    ((100, 0, 256, 16, 1), 1),      # elem_bytes 0: invalid
    ((100, 4, 1, 16, 1), 1),        # k < 2
    ((100, 4, 70000, 16, 1), 1),    # k > 2^16
    ((100, 4, 2048, 16, 1), 2),     # k > device limit
    ((100, 4, 256, 0, 1), 1),       # L = 0
    ((100, 4, 256, 1 << 20, 1), 2), # leaf larger than the smem capacity
])
def test_plan_rejects_out_of_domain(L, args, code):
    assert not L.shuf_plan(*args)
    assert L.shuf_last_status() == code


def test_plan_scratch_and_levels(L):
    p = shuf.shuf_plan(1 << 30, 4, 256, 4096, 1)
    b = p.scratch_bytes
    assert b >= (1 << 30) * 4
    assert b < (1 << 30) * 4 * 1.01  # ping-pong + <= 1 % metadata
    assert p.planned_levels == 3  # 2 expected global levels (SURVEY 8(a) HOT) + 1 spare
    small = shuf.shuf_plan(1000, 4, 256, 4096, 1)
    assert small.planned_levels == 0  # fits one CTA's shared memory
    big = shuf.shuf_plan(1 << 32, 16, 1024, 2048, 11)
    assert big.planned_levels >= 2
    assert big.scratch_bytes >= (1 << 32) * 16


@pytest.mark.parametrize("eb", [1, 2, 3, 12, 32, 64, 256])
def test_gather_route_plans(L, eb):
    """Sizes outside {4, 8, 16} plan the gather route (NEXT-4): the index plan's
    scratch (u32 indices below 2^32 elements) + index array + staging rows."""
    n = 1 << 24
    p = shuf.shuf_plan(n, eb, 256, 4096, 1)
    ix = shuf.shuf_plan(n, 4, 256, 4096, 1)
    assert p.planned_levels == ix.planned_levels
    assert p.scratch_bytes >= ix.scratch_bytes + n * 4 + n * eb
    assert p.scratch_bytes < ix.scratch_bytes + n * 4 + n * eb + 4096
    big = shuf.shuf_plan((1 << 32) + 5, eb, 256, 4096, 1)  # u64 indices
    assert big.scratch_bytes >= ((1 << 32) + 5) * (8 + eb)
    code = L.shuf_aux_bytes_inplace(p.handle, ctypes.byref(ctypes.c_uint64()))
    assert code == 2  # the in-place mode moves 4/8/16-byte elements only


@pytest.mark.parametrize("n,eb,k,L_,bound", [
    (1 << 30, 4, 256, 4096, 0.01),        # HOT
    (1 << 32, 16, 1024, 2048, 0.01),      # config 4
    (1 << 27, 4, 256, 4096, 0.015),       # config 2
    (1 << 20, 4, 256, 4096, 0.02),        # config 1 (4 MiB: the fixed header dominates)
    (1_000_000_007, 8, 256, 2048, 0.035), # config 3: 65536 level-2 segments x 256 buckets of counts
])
def test_scratch_metadata_is_sized_from_the_plan(n, eb, k, L_, bound):
    """shuf_scratch_bytes = the n*eb ping-pong buffer + per-level tables
    sized from the planned recursion, not the worst case."""
    p = shuf.shuf_plan(n, eb, k, L_, 1)
    meta = p.scratch_bytes - n * eb
    assert 0 < meta <= bound * n * eb, (meta, n * eb)


def test_segmented_scratch_covers_the_worst_case():
    """Segment lengths are device data: shuf_segmented's layout assumes every
    level may hold min(num_segments, n/(S_fuse+1)+1) long segments."""
    p = shuf.shuf_plan(1 << 26, 4, 256, 4096, 5)
    one = p.scratch_bytes_segmented(1)
    many = p.scratch_bytes_segmented(65536)
    assert p.scratch_bytes <= one <= many
    assert p.scratch_bytes_segmented(1 << 40) == many or p.scratch_bytes_segmented(1 << 40) >= many


@pytest.mark.parametrize("n,eb,k,L_", [(1 << 30, 4, 256, 4096), (1 << 27, 4, 256, 4096), (1_000_000_007, 8, 256, 2048),
                                        (1 << 32, 16, 1024, 2048), (1 << 20, 4, 256, 4096), (100_000, 4, 2, 1)])
def test_inplace_aux_is_a_small_fraction(n, eb, k, L_):
    """The in-place mode's aux memory is a few percent of
    the data (plus a fixed part for the batch buffers, <= 96 MiB) -- the point
    of the mode -- while the stable mode's scratch holds a full ping-pong copy."""
    p = shuf.shuf_plan(n, eb, k, L_, 1)
    aux = shuf.shuf_aux_bytes_inplace(p)
    assert aux > 0
    assert aux < 0.05 * n * eb + (96 << 20), (aux, n * eb)
    if n * eb >= (1 << 30):
        assert aux < 0.05 * n * eb, (aux, n * eb)
    assert p.scratch_bytes >= n * eb


def test_status_strings(L):
    for c in range(8):
        assert L.shuf_status_string(c)


def test_run_argument_errors_before_any_device_work(L):
    p = shuf.shuf_plan(1000, 4, 64, 100, 1)
    # misaligned pointers are rejected synchronously
    assert L.shuf_run(p.handle, ctypes.c_void_p(0x1004), ctypes.c_void_p(0x2000), 1 << 30, None) == 3
    # scratch too small
    assert L.shuf_run(p.handle, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000), 16, None) == 4
    # n <= 1 is a no-op (nothing enqueued)
    q = shuf.shuf_plan(1, 4, 64, 100, 1)
    assert L.shuf_run(q.handle, ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000), 0, None) == 0


def test_no_oracle_import_in_product_package():
    pkg = os.path.join(ROOT, "paper_2302_03317_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(//|#).*", "", src).lower(), f
