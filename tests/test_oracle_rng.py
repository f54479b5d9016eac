"""Pins for the oracle's random-number layer: D1 Philox,
D4/D5 Lemire.  Every expected value here comes from a library routine or a
closed form, never from the oracle itself."""
import ctypes
import os

import numpy as np
import pytest

import oracle

CURAND_PHILOX = 161  # CURAND_RNG_PSEUDO_PHILOX4_32_10


def test_philox_matches_curand_device_routine_any_counter(curand_ref):
    """D1 vs cuRAND's curand_Philox4x32_10 (host-compiled) on random counters
    and keys, with every counter word (including x1, x3) exercised."""
    rng = np.random.default_rng(20230203)
    N = 4000
    ctr = rng.integers(0, 2**32, size=(N, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(N, 2), dtype=np.uint64).astype(np.uint32)
    # the exact counters D4/D5 use: tags 1..4 in x3, levels/attempts in x2
    ctr[:64, 3] = np.arange(64) % 4 + 1
    ctr[:64, 2] = np.arange(64) | ((np.arange(64) % 3) << 8)
    ctr[64:72] = 0xFFFFFFFF
    key[64:72] = 0xFFFFFFFF
    ref = np.zeros((N, 4), dtype=np.uint32)
    curand_ref.curand_ref_philox(ctr.ctypes.data, key.ctypes.data, ref.ctypes.data, N)
    for i in range(N):
        got = oracle.philox(ctr[i], key[i])
        assert (got == ref[i]).all(), (i, ctr[i], key[i], got, ref[i])


def test_philox_matches_curand_host_generator_stream():
    """D1 vs cuRAND's host generator API (libcurand): in that generator output
    block i is Philox(key=(lo32 seed, hi32 seed), counter=(i>>16, 0, i&0xFFFF, 0))."""
    path = "/usr/local/cuda/lib64/libcurand.so"
    if not os.path.exists(path):
        pytest.skip("libcurand not present")
    cr = ctypes.CDLL(path)
    gen = ctypes.c_void_p()
    assert cr.curandCreateGeneratorHost(ctypes.byref(gen), CURAND_PHILOX) == 0
    try:
        for seed in (0, 1, 7, 0x0123456789ABCDEF):
            assert cr.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
            assert cr.curandSetGeneratorOffset(gen, ctypes.c_ulonglong(0)) == 0
            nblk = 65536 * 2 + 8
            out = np.zeros(nblk * 4, dtype=np.uint32)
            assert cr.curandGenerate(gen, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(out.size)) == 0
            out = out.reshape(-1, 4)
            key = [seed & 0xFFFFFFFF, seed >> 32]
            for i in (0, 1, 2, 5, 65535, 65536, 65537, 131072, 131079):
                ctr = [i >> 16, 0, i & 0xFFFF, 0]
                assert (oracle.philox(ctr, key) == out[i]).all(), (seed, i)
    finally:
        cr.curandDestroyGenerator(gen)


def test_problem_key_is_odd_multiplier_bijection():
    """D2: K(seed, s) = seed + s*gamma mod 2^64; distinct s give distinct keys."""
    g = 0x9E3779B97F4A7C15
    for seed, s in [(0, 0), (5, 1), (5, 65535), (2**64 - 1, 3)]:
        assert oracle.problem_key(seed, s) == (seed + s * g) % 2**64
    keys = {oracle.problem_key(5, s) for s in range(20000)}
    assert len(keys) == 20000


def test_lemire16_exhaustive_all_k(lemire_enum):
    """For EVERY k in [2, 2^16]: each bucket b in [0,k) is hit by exactly
    floor(2^16/k) of the 2^16 words and exactly 2^16 mod k words are rejected
    (Lemire 2019's exactness)."""
    bad = ctypes.c_uint64(0)
    fn = ctypes.cast(oracle.lib().oracle_lemire16_accept, ctypes.c_void_p)
    lemire_enum.lemire16_enumerate(fn, 2, 65536, ctypes.byref(bad))
    assert bad.value == 0


def test_lemire16_power_of_two_is_shift():
    """for s = 2^b the draw is plain shifting (no rejection)."""
    rng = np.random.default_rng(1)
    for b in range(1, 17):
        for v in rng.integers(0, 65536, size=200):
            assert oracle.lemire16(int(v), 1 << b) == int(v) >> (16 - b)


@pytest.mark.parametrize("s", [3, 4095])
def test_lemire32_exhaustive(lemire_enum, s):
    """All 2^32 words for one bound s: every j in [0,s) gets floor(2^32/s)
    words, 2^32 mod s are rejected, and nothing lands outside [0,s)."""
    counts = np.zeros(s + 1, dtype=np.uint64)
    rej = ctypes.c_uint64(0)
    fn = ctypes.cast(oracle.lib().oracle_lemire32_accept, ctypes.c_void_p)
    lemire_enum.lemire32_enumerate(fn, s, counts.ctypes.data, ctypes.byref(rej))
    assert counts[s] == 0
    assert (counts[:s] == 2**32 // s).all()
    assert rej.value == 2**32 % s


def test_lemire32_power_of_two_never_rejects():
    rng = np.random.default_rng(2)
    for b in range(1, 32):
        for w in rng.integers(0, 2**32, size=50, dtype=np.uint64):
            assert oracle.lemire32(int(w), 1 << b) == int(w) >> (32 - b)


def test_bucket_draw_layout_first_principles():
    """D4 lanes for power-of-two k <= 256: the 16 draws of group g are the
    8-bit lanes of Philox(K, (g, level, SC=1)) little-endian, top log2(k)
    bits (shift only); for k > 256 the 8 draws of group g are the
    16-bit lanes of the same counter (level, SC)."""
    K = oracle.problem_key(9, 0)
    key = [K & 0xFFFFFFFF, K >> 32]
    for level in (0, 3):
        for g in (0, 1, 12345, 2**33 + 7):
            w = oracle.philox([g & 0xFFFFFFFF, g >> 32, level, 1], key)
            b8 = [(int(w[j >> 2]) >> (8 * (j & 3))) & 0xFF for j in range(16)]
            assert list(oracle.bucket_draws(K, level, 16 * g, 16, 256)) == b8
            assert list(oracle.bucket_draws(K, level, 16 * g, 16, 64)) == [v >> 2 for v in b8]
            assert list(oracle.bucket_draws(K, level, 16 * g, 16, 2)) == [v >> 7 for v in b8]
            l16 = [(int(w[j >> 1]) >> (16 * (j & 1))) & 0xFFFF for j in range(8)]
            assert list(oracle.bucket_draws(K, level, 8 * g, 8, 1024)) == [v >> 6 for v in l16]
            assert list(oracle.bucket_draws(K, level, 8 * g, 8, 65536)) == l16


def test_bucket_draw_retry_stream():
    """D4 retry: with k=40000 about 39% of words are rejected; a rejected
    position's draw comes from Philox(K, (p, level|(a<<8), SC_RETRY=3)).w0."""
    K = oracle.problem_key(3, 0)
    key = [K & 0xFFFFFFFF, K >> 32]
    k = 40000
    t = 65536 % k
    found = 0
    for p in range(2000):
        b, rej = oracle.bucket_draw(K, 2, p, k)
        g = p >> 3
        w = oracle.philox([g & 0xFFFFFFFF, g >> 32, 2, 1], key)
        v = (int(w[(p & 7) >> 1]) >> (16 * (p & 1))) & 0xFFFF
        a = 0
        while (v * k) & 0xFFFF < t:
            a += 1
            v = int(oracle.philox([p & 0xFFFFFFFF, p >> 32, 2 | (a << 8), 3], key)[0]) & 0xFFFF
        assert rej == a and b == (v * k) >> 16
        found += rej > 0
    assert found > 500


def test_fy_draw_layout_and_retry_16bit():
    """D5, s <= 2^16, keyed by (leaf id q, step i): 16-bit lane i&7 of
    Philox(K, (q, i>>3, FY16=2)); retries from Philox(K, (q, i, 4 | a<<8)).w0
    & 0xFFFF; bound s = i+1 = 40000 rejects ~39% of the lanes."""
    K = oracle.problem_key(11, 2)
    key = [K & 0xFFFFFFFF, K >> 32]
    seen = 0
    for q in (0, 77, 2**40 + 3):
        for i in list(range(1, 200)) + [39999] * 0 + list(range(39990, 40010)):
            s = i + 1
            t = 65536 % s
            j, rej = oracle.fy_draw(K, q, i)
            w = oracle.philox([q & 0xFFFFFFFF, q >> 32, i >> 3, 2], key)
            v = (int(w[(i & 7) >> 1]) >> (16 * (i & 1))) & 0xFFFF
            a = 0
            while (v * s) & 0xFFFF < t:
                a += 1
                v = int(oracle.philox([q & 0xFFFFFFFF, q >> 32, i, 4 | (a << 8)], key)[0]) & 0xFFFF
            assert rej == a and j == (v * s) >> 16 and 0 <= j <= i
            seen += rej > 0
    assert seen > 5


def test_fy_draw_layout_and_retry_32bit():
    """D5, s > 2^16: 32-bit word i&3 of Philox(K, (q, i>>2, FY32=5));
    retries from Philox(K, (q, i, 6 | a<<8)).w0; s=2^31+1 rejects ~half."""
    K = oracle.problem_key(11, 2)
    key = [K & 0xFFFFFFFF, K >> 32]
    seen = 0
    for q in (0, 5, 2**40 + 3):
        for i in list(range(2**31, 2**31 + 100)) + [70000, 65536]:
            s = i + 1
            t = 2**32 % s
            j, rej = oracle.fy_draw(K, q, i)
            w = int(oracle.philox([q & 0xFFFFFFFF, q >> 32, i >> 2, 5], key)[i & 3])
            a = 0
            while (w * s) % 2**32 < t:
                a += 1
                w = int(oracle.philox([q & 0xFFFFFFFF, q >> 32, i, 6 | (a << 8)], key)[0])
            assert rej == a and j == (w * s) >> 32 and 0 <= j <= i
            seen += rej > 0
    assert seen > 50


def test_fy_draw_boundary_65535_uses_16bit_lanes():
    """i = 65535 (s = 2^16): 16-bit lanes, pure shift, no rejection."""
    K = oracle.problem_key(1, 0)
    key = [K & 0xFFFFFFFF, K >> 32]
    for q in range(8):
        i = 65535
        w = oracle.philox([q, 0, i >> 3, 2], key)
        v = (int(w[(i & 7) >> 1]) >> (16 * (i & 1))) & 0xFFFF
        assert oracle.fy_draw(K, q, i) == (v, 0)
