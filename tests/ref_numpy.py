"""A second, independent re-derivation of DESIGN.md's definition in numpy
(SURVEY B3).  It is written level-by-level (breadth first, as D6 is stated)
while the C oracle recurses depth first (Fig. 2), and it draws with a
vectorised numpy Philox instead of the oracle's.  Agreement of the two on
small inputs catches layout slips in either; it is a cross-check, not a pin
(both read the same definition), so the pins live in test_oracle_*.py."""
from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)


def philox_np(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10 over arrays of counter words (uint64 holding u32)."""
    x0, x1, x2, x3 = (np.asarray(c, dtype=np.uint64) & M32 for c in (c0, c1, c2, c3))
    x0, x1, x2, x3 = np.broadcast_arrays(x0, x1, x2, x3)
    ka, kb = np.uint64(k0), np.uint64(k1)
    for r in range(10):
        if r:
            ka = (ka + np.uint64(0x9E3779B9)) & M32
            kb = (kb + np.uint64(0xBB67AE85)) & M32
        p0 = x0 * np.uint64(0xD2511F53)
        p1 = x2 * np.uint64(0xCD9E8D57)
        x0, x1, x2, x3 = ((p1 >> np.uint64(32)) ^ x1 ^ ka, p1 & M32, (p0 >> np.uint64(32)) ^ x3 ^ kb, p0 & M32)
    return x0, x1, x2, x3


def _narrow_shift(k: int):
    return (k.bit_length() - 1) if (k <= 256 and k & (k - 1) == 0) else -1


def bucket_np(K: int, level: int, p: np.ndarray, k: int) -> np.ndarray:
    p = np.asarray(p, dtype=np.uint64)
    kw = (K & 0xFFFFFFFF, K >> 32)
    b = _narrow_shift(k)
    if b >= 0:
        g = p >> np.uint64(4)
        W = np.stack(philox_np(g & M32, g >> np.uint64(32), np.uint64(level), np.uint64(1), *kw))
        j = (p & np.uint64(15)).astype(np.int64)
        word = W[j >> 2, np.arange(p.shape[0])]
        v = (word >> (np.uint64(8) * (j & 3).astype(np.uint64))) & np.uint64(0xFF)
        return (v >> np.uint64(8 - b)).astype(np.int64)
    g = p >> np.uint64(3)
    W = np.stack(philox_np(g & M32, g >> np.uint64(32), np.uint64(level), np.uint64(1), *kw))
    j = (p & np.uint64(7)).astype(np.int64)
    word = W[j >> 1, np.arange(p.shape[0])]
    v = (word >> (np.uint64(16) * (j & 1).astype(np.uint64))) & np.uint64(0xFFFF)
    t = np.uint64(65536 % k)
    m = v * np.uint64(k)
    out = (m >> np.uint64(16)).astype(np.int64)
    bad = (m & np.uint64(0xFFFF)) < t
    a = 0
    while bad.any():
        a += 1
        pb = p[bad]
        w0 = philox_np(pb & M32, pb >> np.uint64(32), np.uint64(level | (a << 8)), np.uint64(3), *kw)[0]
        mb = (w0 & np.uint64(0xFFFF)) * np.uint64(k)
        idx = np.nonzero(bad)[0]
        ok = (mb & np.uint64(0xFFFF)) >= t
        out[idx[ok]] = (mb[ok] >> np.uint64(16)).astype(np.int64)
        bad[idx[ok]] = False
    return out


def fy_np(K: int, q: int, i: np.ndarray) -> np.ndarray:
    """D5 for steps i (bound i+1 <= 2^16) of the leaf starting at position q."""
    i = np.asarray(i, dtype=np.uint64)
    s = i + np.uint64(1)
    assert (s <= 65536).all()
    kw = (K & 0xFFFFFFFF, K >> 32)
    q = np.uint64(q)
    W = np.stack(philox_np(q & M32, q >> np.uint64(32), i >> np.uint64(3), np.uint64(2), *kw))
    j = (i & np.uint64(7)).astype(np.int64)
    v = (W[j >> 1, np.arange(i.shape[0])] >> (np.uint64(16) * (j & 1).astype(np.uint64))) & np.uint64(0xFFFF)
    t = np.uint64(65536) % s
    out = np.zeros(i.shape[0], dtype=np.int64)
    todo = np.ones(i.shape[0], dtype=bool)
    a = 0
    while todo.any():
        idx = np.nonzero(todo)[0]
        if a:
            v_i = philox_np(q & M32, q >> np.uint64(32), i[idx], np.uint64(4 | (a << 8)), *kw)[0] & np.uint64(0xFFFF)
        else:
            v_i = v[idx]
        m = v_i * s[idx]
        ok = (m & np.uint64(0xFFFF)) >= t[idx]
        out[idx[ok]] = (m[ok] >> np.uint64(16)).astype(np.int64)
        todo[idx[ok]] = False
        a += 1
    return out


def shuffle_np(data: np.ndarray, k: int, L: int, K: int, max_levels: int = 1 << 30, run_leaves: bool = True):
    """D6 breadth first: segs_l -> stable scatter -> children; FY on leaves last."""
    A = np.array(data, copy=True)
    n = A.shape[0]
    leaves = []
    segs = [(0, n)] if n > L else []
    if n <= L:
        leaves.append((0, n))
    level = 0
    while segs and level < max_levels:
        nxt = []
        for a, m in segs:
            pos = np.arange(a, a + m, dtype=np.uint64)
            b = bucket_np(K, level, pos, k)
            order = np.argsort(b, kind="stable")
            A[a:a + m] = A[a:a + m][order]
            cnt = np.bincount(b, minlength=k)
            start = a
            for c in cnt:
                (nxt if c > L else leaves).append((start, int(c)))
                start += int(c)
        segs = nxt
        level += 1
    if run_leaves:
        for q, m in leaves:
            if m < 2:
                continue
            i = np.arange(m - 1, 0, -1)
            j = fy_np(K, q, i)
            for ii, jj in zip(i, j):
                A[[q + ii, q + jj]] = A[[q + jj, q + ii]]
    return A
