"""CPU oracle for the deterministic ScatterShuffle definition.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2302_03317_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``shuf_oracle.c`` (plain single-threaded C, one
function per definition step, each citing PAPER.md); this module only
marshals numpy arrays through ctypes.  ``build()`` compiles the C file with
gcc into ``liboracle.so`` next to it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "shuf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ERR_INVALID_ARG = 1
ERR_DEPTH = 5
ERR_NOMEM = 7
ALL_LEVELS = 0xFFFFFFFF


class Stats(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_uint32),
        ("pad", ctypes.c_uint32),
        ("scatter_elems", ctypes.c_uint64 * 257),
        ("leaves", ctypes.c_uint64),
        ("bucket_rejections", ctypes.c_uint64),
        ("fy_rejections", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {
            "levels": int(self.levels),
            "scatter_elems": [int(self.scatter_elems[i]) for i in range(self.levels)],
            "leaves": int(self.leaves),
            "bucket_rejections": int(self.bucket_rejections),
            "fy_rejections": int(self.fy_rejections),
        }


def build(force: bool = False) -> str:
    """Compile shuf_oracle.c -> liboracle.so (gcc, -O2, no -ffast-math)."""
    hdr = os.path.join(_HERE, "shuf_oracle.h")
    stale = (not os.path.exists(_LIB)) or max(os.path.getmtime(_SRC), os.path.getmtime(hdr)) > os.path.getmtime(_LIB)
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32, u64, vp, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
        L.oracle_problem_key.argtypes = [u64, u64]
        L.oracle_problem_key.restype = u64
        L.oracle_lemire16_accept.argtypes = [u32, u32, vp]
        L.oracle_lemire16_accept.restype = i32
        L.oracle_lemire32_accept.argtypes = [u32, u32, vp]
        L.oracle_lemire32_accept.restype = i32
        L.oracle_bucket_draw.argtypes = [u64, u32, u64, u32, vp]
        L.oracle_bucket_draw.restype = u32
        L.oracle_fy_draw.argtypes = [u64, u64, u32, vp]
        L.oracle_fy_draw.restype = u32
        L.oracle_bucket_draws.argtypes = [u64, u32, u64, u64, u32, vp]
        L.oracle_fy_draws.argtypes = [u64, vp, vp, u64, vp]
        L.oracle_fy_with_draws.argtypes = [vp, u64, u32, vp]
        L.oracle_shuffle.argtypes = [vp, u64, u32, u32, u32, u64, u32, i32, vp]
        L.oracle_shuffle.restype = i32
        L.oracle_segmented.argtypes = [vp, vp, u64, u32, u32, u32, u64, u32, i32, vp]
        L.oracle_segmented.restype = i32
        L.oracle_points.argtypes = [u64, u32, u32, u64, vp, u64, vp]
        L.oracle_points.restype = i32
        L.oracle_sim_rough_scatter.argtypes = [u64, u32, u64, u32, vp, vp]
        L.oracle_sim_rough_scatter.restype = i32
        L.oracle_ipsc_draw.argtypes = [u64, u32, u32, u32, u32, u64, u32]
        L.oracle_ipsc_draw.restype = u32
        L.oracle_ipsc_depth.argtypes = [u64, u32]
        L.oracle_ipsc_depth.restype = u32
        L.oracle_ipsc_shuffle.argtypes = [vp, u64, u32, u32, u32, u64, u32, i32, vp, vp]
        L.oracle_ipsc_shuffle.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def philox(ctr, key):
    """D1: Philox4x32-10 of one 128-bit counter under a 64-bit key (4 + 2 u32 words)."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def problem_key(seed: int, s: int) -> int:
    """D2: K(seed, s) = seed + s * 0x9E3779B97F4A7C15 mod 2^64."""
    return int(lib().oracle_problem_key(seed, s))


def lemire16(v: int, k: int):
    out = ctypes.c_uint32()
    ok = lib().oracle_lemire16_accept(v, k, ctypes.byref(out))
    return int(out.value) if ok else None


def lemire32(w: int, s: int):
    out = ctypes.c_uint32()
    ok = lib().oracle_lemire32_accept(w, s, ctypes.byref(out))
    return int(out.value) if ok else None


def bucket_draw(K: int, level: int, p: int, k: int):
    """D4 for one position; returns (bucket, retries)."""
    rej = ctypes.c_uint64(0)
    b = lib().oracle_bucket_draw(K, level, p, k, ctypes.byref(rej))
    return int(b), int(rej.value)


def fy_draw(K: int, q: int, i: int):
    """D5 for step i (bound i+1) of the leaf starting at problem position q;
    returns (partner, retries)."""
    rej = ctypes.c_uint64(0)
    j = lib().oracle_fy_draw(K, q, i, ctypes.byref(rej))
    return int(j), int(rej.value)


def bucket_draws(K: int, level: int, p0: int, count: int, k: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint32)
    lib().oracle_bucket_draws(K, level, p0, count, k, _ptr(out))
    return out


def fy_draws(K: int, q, i) -> np.ndarray:
    """D5 for arrays of (leaf start q, step i)."""
    q = np.ascontiguousarray(np.broadcast_to(np.asarray(q, dtype=np.uint64), np.shape(i)))
    i = np.ascontiguousarray(i, dtype=np.uint32)
    out = np.zeros(i.shape[0], dtype=np.uint32)
    lib().oracle_fy_draws(K, _ptr(q), _ptr(i), i.shape[0], _ptr(out))
    return out


def fy_with_draws(data: np.ndarray, j) -> np.ndarray:
    """Fig. 1 loop with the partner draws given explicitly (stub generator)."""
    a = np.ascontiguousarray(data).copy()
    jj = np.ascontiguousarray(j, dtype=np.uint32)
    assert jj.shape[0] >= a.shape[0]
    lib().oracle_fy_with_draws(_ptr(a), a.shape[0], a.dtype.itemsize if a.ndim == 1 else a.strides[0], _ptr(jj))
    return a


def _elem_bytes(a: np.ndarray) -> int:
    return a.strides[0] if a.ndim > 1 else a.dtype.itemsize


def shuffle(data: np.ndarray, k: int, L: int, seed: int, max_levels: int = ALL_LEVELS,
            run_leaves: bool = True, inplace: bool = False, stats: bool = False):
    """D6: the whole deterministic ScatterShuffle of ``data`` (rows are elements)."""
    a = data if inplace else np.ascontiguousarray(data).copy()
    assert a.flags["C_CONTIGUOUS"]
    st = Stats()
    rc = lib().oracle_shuffle(_ptr(a), a.shape[0], _elem_bytes(a), k, L, seed, max_levels,
                              1 if run_leaves else 0, ctypes.byref(st))
    if rc:
        raise RuntimeError(f"oracle_shuffle failed with status {rc}")
    return (a, st.as_dict()) if stats else a


def segmented(data: np.ndarray, offsets, k: int, L: int, seed: int, max_levels: int = ALL_LEVELS,
              run_leaves: bool = True, inplace: bool = False, stats: bool = False):
    """D7: independent D6 per segment [offsets[s], offsets[s+1]) with key K(seed, s)."""
    a = data if inplace else np.ascontiguousarray(data).copy()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    st = Stats()
    rc = lib().oracle_segmented(_ptr(a), _ptr(off), off.shape[0] - 1, _elem_bytes(a), k, L, seed, max_levels,
                                1 if run_leaves else 0, ctypes.byref(st))
    if rc:
        raise RuntimeError(f"oracle_segmented failed with status {rc}")
    return (a, st.as_dict()) if stats else a


def points(n: int, k: int, L: int, seed: int, js) -> np.ndarray:
    """D6 point queries: pi(j) = input index of the element at output position j
    of the single shuffle of n elements (key K = seed), for each j in ``js``,
    without materialising the array (for sampled checks at full size).  For a
    segment s of a batch pass seed = K(seed, s) and segment-relative j."""
    j = np.ascontiguousarray(js, dtype=np.uint64)
    out = np.zeros(j.shape[0], dtype=np.uint64)
    rc = lib().oracle_points(n, k, L, seed, _ptr(j), j.shape[0], _ptr(out))
    if rc:
        raise RuntimeError(f"oracle_points failed with status {rc}")
    return out


def sim_rough_scatter(n: int, k: int, seed: int, runs: int):
    """D9 (NEXT-1): per run r (key K(seed, r)) the RoughScatter stop
    time T (items placed when the first bucket fills, Lemma 2: R = n - T) and
    the TwoSweep swap count M = sum_i |D_i| (Lemma 4).  Returns (T, M)."""
    T = np.zeros(runs, dtype=np.uint64)
    M = np.zeros(runs, dtype=np.uint64)
    rc = lib().oracle_sim_rough_scatter(n, k, seed, runs, _ptr(T), _ptr(M))
    if rc:
        raise RuntimeError(f"oracle_sim_rough_scatter failed with status {rc}")
    return T, M


class IpscStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in
                ("segments", "rough_steps", "merge_swaps", "staged", "transfers", "dsum", "leaves")]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


IPSC_RS, IPSC_FM, IPSC_FY = 7, 8, 9


def ipsc_draw(K: int, tag: int, c0: int, c1: int, level: int, a: int, bound: int) -> int:
    """D10 draw: first Lemire32-accepted word of Philox(K, (c0, c1, lo32 a,
    tag | level << 8 | (hi32 a & 0xFFFF) << 16)) for the bound."""
    return int(lib().oracle_ipsc_draw(K, tag, c0, c1, level, a, bound))


def ipsc_depth(m: int, k: int) -> int:
    """D10: ParRoughScatter tree depth t = min(11, floor(log2(m / k^2)))."""
    return int(lib().oracle_ipsc_depth(m, k))


def ipsc_shuffle(data: np.ndarray, k: int, L: int, seed: int, max_levels: int = ALL_LEVELS,
                 run_leaves: bool = True, stats: bool = False):
    """D10 (NEXT-2): the paper's In-Place ScatterShuffle (P:150-265, P:322-425,
    P:479-491) with deterministic counter-based draws.  Returns the shuffled
    copy, and with stats=True also (stats dict, level-0 final bucket sizes)."""
    a = np.ascontiguousarray(data).copy()
    st = IpscStats()
    sizes0 = np.zeros(k, dtype=np.uint64)
    rc = lib().oracle_ipsc_shuffle(_ptr(a), a.shape[0], _elem_bytes(a), k, L, seed, max_levels,
                                   1 if run_leaves else 0, ctypes.byref(st), _ptr(sizes0))
    if rc:
        raise RuntimeError(f"oracle_ipsc_shuffle failed with status {rc}")
    return (a, st.as_dict(), sizes0) if stats else a
