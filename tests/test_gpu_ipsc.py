"""GPU parity of the paper's In-Place ScatterShuffle (SURVEY 8(f) NEXT-2,
DESIGN.md D10, kernels_ipsc.cu): RoughScatter in
ParRoughScatter's split/merge tree, FineScatter's multinomial
sizes, TwoSweep and stash shuffle, recursively (Fig. 2) with
Fisher-Yates leaves -- against oracle.ipsc_shuffle, element by element, bit
for bit (integer work), whole runs and level-limited runs."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2302_03317_b200 as shuf  # noqa: E402
from tests.gpu_util import to_dev, to_host  # noqa: E402


def _input(n, eb, seed):
    rng = np.random.default_rng(seed)
    if eb == 4:
        return np.arange(n, dtype=np.uint32)
    if eb == 8:
        return rng.integers(0, 2**63, size=n, dtype=np.uint64)
    a = np.empty((n, 2), dtype=np.uint64)
    a[:, 0] = np.arange(n, dtype=np.uint64)
    a[:, 1] = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    return a


def _gpu(a, k, L, seed, eb, max_levels=None, run_leaves=True):
    x = to_dev(a)
    shuf.ipsc_shuffle(x, k, L, seed, elem_bytes=eb, max_levels=max_levels, run_leaves=run_leaves)
    return to_host(x, a)


LEVEL1 = [
    # n, k, L, seed, eb: one IpSc level (no leaves) -- RoughScatter tree + FineScatter
    (1000, 4, 16, 1, 4),           # t = 5 (m / k^2 = 62)
    (5000, 16, 64, 2, 4),          # t = 4
    (65_537, 16, 64, 3, 4),        # t = 8
    (200_003, 256, 300, 4, 4),     # t = 1
    (50_000, 3, 5, 5, 4),          # non-power-of-two k, t = 11
    (30_000, 1000, 40, 6, 4),      # k^2 > m: t = 0, buckets of 30
    (3_000_000, 256, 4096, 7, 4),  # t = 5
    (300_007, 64, 128, 8, 8),      # u64
    (100_003, 128, 64, 9, 16),     # 16-byte records
    (20, 7, 1, 10, 4),             # tiny
]


@pytest.mark.parametrize("n,k,L,seed,eb", LEVEL1)
def test_ipsc_one_level_equals_oracle(n, k, L, seed, eb):
    a = _input(n, eb, seed)
    got = _gpu(a, k, L, seed, eb, max_levels=1, run_leaves=False)
    exp = oracle.ipsc_shuffle(a, k, L, seed, max_levels=1, run_leaves=False)
    assert (got == exp).all()


FULL = [
    (2, 2, 1, 1, 4), (3, 2, 1, 2, 4), (1000, 256, 4096, 3, 4),   # root leaf
    (4097, 256, 4096, 4, 4),
    (65_537, 16, 64, 5, 4),
    (200_003, 256, 300, 6, 4),
    (50_000, 3, 5, 7, 4),
    (30_000, 1000, 40, 8, 4),
    (1_000_003, 256, 4096, 9, 4),
    (4_000_037, 256, 2048, 10, 8),
    (500_000, 1024, 2048, 11, 16),
    (20_000_003, 256, 2048, 3, 8),      # config-3 shape (u64, L = 2048), three IpSc levels
    (8_000_000, 1024, 2048, 11, 16),    # config-4 shape (16-byte records, k = 1024)
]


@pytest.mark.parametrize("n,k,L,seed,eb", FULL)
def test_ipsc_whole_shuffle_equals_oracle(n, k, L, seed, eb):
    a = _input(n, eb, seed)
    got = _gpu(a, k, L, seed, eb)
    exp = oracle.ipsc_shuffle(a, k, L, seed)
    assert (got == exp).all()


def test_ipsc_two_levels_equal_oracle():
    n, k, L, seed = 2_000_000, 64, 256, 12
    a = _input(n, 4, seed)
    got = _gpu(a, k, L, seed, 4, max_levels=2, run_leaves=False)
    exp = oracle.ipsc_shuffle(a, k, L, seed, max_levels=2, run_leaves=False)
    assert (got == exp).all()


def test_ipsc_aux_is_small():
    """O(k * subtasks) words plus the segment lists: a few percent of the data at most."""
    for n, eb, k, L in [(1 << 30, 4, 256, 4096), (1_000_000_007, 8, 256, 2048), (1 << 32, 16, 1024, 2048)]:
        plan = shuf.shuf_plan(n, eb, k, L, 1)
        assert shuf.shuf_aux_bytes_ipsc(plan) < 0.02 * n * eb


@pytest.mark.parametrize("n,k,L,seed,eb", [(65_537, 16, 64, 5, 4), (1_000_003, 256, 4096, 9, 4),
                                           (300_007, 64, 128, 8, 8), (50_000, 3, 5, 7, 4)])
def test_ipsc_hbm_route_equals_oracle(n, k, L, seed, eb, monkeypatch):
    """Every segment through the HBM kernels (no shared-memory fused level)."""
    monkeypatch.setenv("SHUF_IPSC_NOSMALL", "1")
    a = _input(n, eb, seed)
    assert (_gpu(a, k, L, seed, eb) == oracle.ipsc_shuffle(a, k, L, seed)).all()
