"""GPU parity of the sharded single shuffle (NEXT-3, SURVEY 8(e);
paper_2302_03317_b200/sharded.py): all G ranks run on this one GPU one after
another (no rank waits on another's kernels), each through the C ABI
(shuf_shard_scatter -> exchange layout -> shuf_shard_continue), and the
concatenated output must equal the oracle's D6 of the WHOLE array bit for bit
(P:140-142 level 0 + Fig. 1 leaves, D6)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2302_03317_b200 import sharded  # noqa: E402
from tests.gpu_util import to_dev  # noqa: E402


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


CASES = [
    # n, k, L, seed, eb, world
    (1000, 256, 4096, 3, 4, 2),          # n <= L: one leaf, gathered to rank 0
    (4097, 256, 4096, 4, 4, 2),          # just above L: level 0 on slices shorter than L
    (5000, 256, 4096, 5, 4, 3),
    (300_001, 256, 4096, 7, 4, 3),       # children are leaves
    (3_000_000, 256, 4096, 11, 4, 4),    # children take an in-smem level (finish)
    (20_000_000, 256, 4096, 13, 4, 2),   # children exceed the fused size: an HBM level 1
    (2_000_003, 7, 64, 19, 8, 3),        # non-power-of-two k, u64
    (1_000_000, 1024, 2048, 11, 16, 8),  # 16-byte records, k = 1024 (config-4 shape)
    (1_500_000, 2, 4096, 23, 4, 2),      # k = 2: each rank owns one bucket
    (777_777, 256, 4096, 29, 4, 1),      # one rank: the exchange is local copies
]


@pytest.mark.parametrize("n,k,L,seed,eb,world", CASES)
def test_sharded_equals_oracle(n, k, L, seed, eb, world):
    a = _input(n, eb, seed)
    out, parts = sharded.simulate_sharded(to_dev(a), n, world, k, L, seed, elem_bytes=eb)
    got = out.cpu().numpy().view(a.dtype).reshape(a.shape)
    exp = oracle.shuffle(a, k, L, seed)
    assert (got == exp).all()
    at = 0
    for base, m in parts:
        assert base == at
        at += m
    assert at == n


def test_shard_scatter_is_oracle_level0_of_the_slice():
    """Step 1 alone: rank r's grouped slice and counts (D4 at global positions)."""
    import paper_2302_03317_b200 as shuf
    n, k, L, seed, world = 2_500_000, 256, 4096, 31, 3
    a = _input(n, 4, seed)
    for r in range(world):
        st = sharded.ShardedShuffle(n, 4, k, L, seed, r, world)
        x = to_dev(a[st.lo:st.hi])
        st.scatter(x)
        assert shuf.shuf_last_device_error(st.plan) == 0
        ids = oracle.bucket_draws(oracle.problem_key(seed, 0), 0, st.lo, st.hi - st.lo, k)
        exp = a[st.lo:st.hi][np.argsort(ids, kind="stable")]
        got = st.send[: (st.hi - st.lo) * 4].cpu().numpy().view(np.uint32)
        assert (got == exp).all()
        assert (st.counts.cpu().numpy() == np.bincount(ids, minlength=k)).all()


def test_sharded_repeated_steps_reuse_buffers():
    """The same rank states run twice (bench reuse): identical results."""
    n, k, L, seed, world = 1_200_000, 256, 4096, 37, 2
    a = _input(n, 4, seed)
    sts = [sharded.ShardedShuffle(n, 4, k, L, seed, r, world) for r in range(world)]
    o1, _ = sharded.simulate_sharded(to_dev(a), n, world, k, L, seed, states=sts)
    o2, _ = sharded.simulate_sharded(to_dev(a), n, world, k, L, seed, states=sts)
    assert torch.equal(o1, o2)
    assert (o1.cpu().numpy().view(np.uint32) == oracle.shuffle(a, k, L, seed)).all()
