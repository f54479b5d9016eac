"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the shuffle's arithmetic (no Philox, no Lemire, no
scatter): only the workload generators of BASELINE.json's configs and the
SplitMix64 input generator they name (reading Q10).
Both numpy (host) and torch (host or device) versions are given; a test pins
them equal.

SplitMix64 (Steele, Lea, Flood 2014): state += GAMMA; z = state;
z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB;
return z ^ z>>31.  ``mix64`` is that finaliser.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


# ----------------------------------------------------------------- numpy --
def mix64_np(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def splitmix64_stream_np(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start .. start+count-1 of a SplitMix64 generator seeded with ``seed``
    (output i = mix64(seed + (i+1)*GAMMA))."""
    i = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + (i + np.uint64(1)) * np.uint64(GAMMA)
    return mix64_np(st)


def splitmix64_of_np(x: np.ndarray) -> np.ndarray:
    """splitmix64(x) := first output of a generator seeded with x = mix64(x + GAMMA)."""
    with np.errstate(over="ignore"):
        return mix64_np(np.asarray(x, dtype=np.uint64) + np.uint64(GAMMA))


# ----------------------------------------------------------------- torch --
def _srl(t, s: int):
    """Logical right shift of an int64 tensor holding u64 bits."""
    import torch
    return (t >> s) & ((1 << (64 - s)) - 1)


def _u64_const(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def mix64_torch(z):
    z = (z ^ _srl(z, 30)) * _u64_const(_M1)
    z = (z ^ _srl(z, 27)) * _u64_const(_M2)
    return z ^ _srl(z, 31)


def splitmix64_stream_torch(seed: int, start: int, count: int, device="cpu"):
    import torch
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    st = i * _u64_const(GAMMA) + _u64_const(seed)
    return mix64_torch(st)


def splitmix64_of_torch(x):
    return mix64_torch(x + _u64_const(GAMMA))


# ------------------------------------------------------------- workloads --
@dataclass
class Workload:
    """One BASELINE.json config (or the HOT run of SURVEY 8(c) Q12)."""
    name: str
    n: int
    elem_bytes: int
    k: int
    L: int
    seed: int
    kind: str                      # "iota32" | "splitmix64" | "records" | "segmented"
    num_segments: int = 0
    note: str = ""
    extra: dict = field(default_factory=dict)


WORKLOADS = {
    "c1": Workload("c1", 1 << 20, 4, 256, 4096, 1, "iota32", note="2^20 u32 iota"),
    "c2": Workload("c2", 1 << 27, 4, 256, 4096, 7, "iota32", note="2^27 u32 iota"),
    "c3": Workload("c3", 1_000_000_007, 8, 256, 2048, 3, "splitmix64",
                   note="u64 = outputs of SplitMix64(seed=3)"),
    "c4": Workload("c4", 1 << 32, 16, 1024, 2048, 11, "records",
                   note="16-B records {key=i, payload=splitmix64(i)}"),
    "c5": Workload("c5", 0, 4, 64, 4096, 5, "segmented", num_segments=65536,
                   note="65536 segments, len U[1000,4000] from SplitMix64(seed=5), u32 in-segment iota"),
    "hot": Workload("hot", 1 << 30, 4, 256, 4096, 1, "iota32", note="2^30 u32 iota (the metric's run)"),
}


def c5_lengths(num_segments: int = 65536, seed: int = 5) -> np.ndarray:
    """len_s = 1000 + floor(x_s * 3001 / 2^64), x_s = output s of SplitMix64(seed)."""
    x = splitmix64_stream_np(seed, 0, num_segments)
    hi = (x >> np.uint64(32)).astype(np.uint64)
    lo = (x & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    # floor(x*3001 / 2^64) computed exactly with 32-bit halves
    t = (lo * np.uint64(3001)) >> np.uint64(32)
    lens = (hi * np.uint64(3001) + t) >> np.uint64(32)
    return (lens + np.uint64(1000)).astype(np.int64)


def segment_offsets(lengths: np.ndarray) -> np.ndarray:
    off = np.zeros(lengths.shape[0] + 1, dtype=np.uint64)
    np.cumsum(lengths, out=off[1:])
    return off


def make_input_np(w: Workload, n: int | None = None, offsets: np.ndarray | None = None) -> np.ndarray:
    """Host (numpy) input for workload ``w``; ``n`` overrides the size (bounded samples)."""
    n = w.n if n is None else n
    if w.kind == "iota32":
        return np.arange(n, dtype=np.uint32)
    if w.kind == "splitmix64":
        return splitmix64_stream_np(w.seed, 0, n)
    if w.kind == "records":
        rec = np.empty((n, 2), dtype=np.uint64)
        rec[:, 0] = np.arange(n, dtype=np.uint64)
        rec[:, 1] = splitmix64_of_np(rec[:, 0])
        return rec
    if w.kind == "segmented":
        assert offsets is not None
        lens = np.diff(offsets.astype(np.int64))
        starts = np.repeat(offsets[:-1].astype(np.int64), lens)
        return (np.arange(int(offsets[-1]), dtype=np.int64) - starts).astype(np.uint32)
    raise ValueError(w.kind)


def make_input_torch(w: Workload, device, n: int | None = None, offsets=None):
    """Device (torch) input for workload ``w`` with the same bits as make_input_np."""
    import torch
    n = w.n if n is None else n
    if w.kind == "iota32":
        # u32 bits carried in an int32 tensor
        return torch.arange(n, dtype=torch.int64, device=device).to(torch.int32) if n < (1 << 31) else \
            (torch.arange(n, dtype=torch.int64, device=device) & 0xFFFFFFFF).to(torch.int32)
    if w.kind == "splitmix64":
        return splitmix64_stream_torch(w.seed, 0, n, device=device)
    if w.kind == "records":
        rec = torch.empty((n, 2), dtype=torch.int64, device=device)
        step = 1 << 28
        for s in range(0, n, step):
            e = min(n, s + step)
            idx = torch.arange(s, e, dtype=torch.int64, device=device)
            rec[s:e, 0] = idx
            rec[s:e, 1] = splitmix64_of_torch(idx)
        return rec
    if w.kind == "segmented":
        off = torch.as_tensor(np.asarray(offsets, dtype=np.int64), device=device)
        lens = off[1:] - off[:-1]
        starts = torch.repeat_interleave(off[:-1], lens)
        return (torch.arange(int(off[-1]), dtype=torch.int64, device=device) - starts).to(torch.int32)
    raise ValueError(w.kind)
