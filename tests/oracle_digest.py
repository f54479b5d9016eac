"""Whole-array oracle results for the full-size parity tests, computed in
worker processes (one host core each) while the GPU side runs.

TEST INFRASTRUCTURE: imports oracle/ (allowed in tests/ only).  A worker
returns per-chunk BLAKE2b digests of the oracle's output instead of the
array itself (4-16 GB would not pass cheaply between processes); the test
digests the GPU output the same way, so equal digest lists mean equal arrays
(up to a 2^-128 collision), and a differing chunk is named.

Jobs (BASELINE.json configs at full size):
- ``hot``: 2^30 u32 iota, k=256, L=4096, seed=1 (the metric's run);
- ``c3``:  1,000,000,007 SplitMix64(3) u64 values, k=256, L=2048, seed=3;
- ``hot_ipsc``: HOT through the paper's In-Place ScatterShuffle (D10, NEXT-2);
- ``c4pi``: the permutation pi of config 4 (2^32 elements, k=1024, L=2048,
  seed=11) computed on u32 iota -- pi does not depend on the element size
  (D6), so the GPU's 16-byte records must carry key[j] = pi(j)
  (SURVEY 8(c) "Config-4 check").  ~40 GB of host RAM, a few minutes.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

CHUNK = 1 << 24  # elements per digest


def digests(arr: np.ndarray) -> list:
    """Per-chunk digests of a 1-D array's bytes (CHUNK elements per chunk)."""
    out = []
    for s in range(0, arr.shape[0], CHUNK):
        out.append(hashlib.blake2b(np.ascontiguousarray(arr[s:s + CHUNK]).tobytes(), digest_size=16).hexdigest())
    return out


def job(name: str, n: int | None = None) -> list:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import oracle
    import synth
    if name == "c4pi":
        w = synth.WORKLOADS["c4"]
        a = np.arange(w.n if n is None else n, dtype=np.uint32)
    elif name == "hot_ipsc":
        w = synth.WORKLOADS["hot"]
        return digests(oracle.ipsc_shuffle(synth.make_input_np(w, n=n), w.k, w.L, w.seed))
    else:
        w = synth.WORKLOADS[name]
        a = synth.make_input_np(w, n=n)
    oracle.shuffle(a, w.k, w.L, w.seed, inplace=True)
    return digests(a)


def first_mismatch(got: list, exp: list):
    """Index of the first differing chunk (None if the lists are equal)."""
    if len(got) != len(exp):
        return min(len(got), len(exp))
    for i, (g, e) in enumerate(zip(got, exp)):
        if g != e:
            return i
    return None
