"""NEXT-3 host logic (paper_2302_03317_b200/sharded.py) on CPU: the exchange
layout of the sharded single shuffle, and a world-size-2 gloo run of the
real exchange (torch.distributed p2p) whose level-0 grouping and final
pieces come from the oracle -- the data path itself is the GPU kernels
(tests/test_gpu_sharded.py).  Pins: after the exchange every rank holds
exactly the oracle's level-0 output (D6 with max_levels = 1) at
its global range, and the ranks' ranges tile [0, N)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2302_03317_b200 import sharded  # noqa: E402


@pytest.mark.parametrize("world,k", [(1, 4), (2, 2), (2, 256), (3, 7), (4, 256), (8, 1024), (5, 16)])
def test_exchange_plan_tiles_and_pairs(world, k):
    rng = np.random.default_rng(world * 1000 + k)
    counts = rng.integers(0, 50, size=(world, k)).tolist()
    counts[0][0] = 0
    exs = [sharded.exchange_plan(counts, world, k, r) for r in range(world)]
    N = int(np.sum(counts))
    # the owned output ranges tile [0, N) in rank order
    at = 0
    for ex in exs:
        assert ex.base == at
        assert ex.child_offsets[0] == 0 and ex.child_offsets[-1] == ex.m
        assert all(a <= b for a, b in zip(ex.child_offsets, ex.child_offsets[1:]))
        at += ex.m
    assert at == N
    # every (source, bucket) piece leaves once and arrives once, same length, same order per pair
    for r, ex in enumerate(exs):
        cover = np.zeros(ex.m, dtype=np.int64)
        for (_, at, c) in ex.local:
            cover[at:at + c] += 1
        for (_, at, c) in ex.recvs:
            cover[at:at + c] += 1
        assert (cover == 1).all()
        sent = sum(c for _, _, c in ex.sends) + sum(c for _, _, c in ex.local)
        assert sent == sum(counts[r])
    for s in range(world):
        for d in range(world):
            if s == d:
                continue
            out = [c for (p, _, c) in exs[s].sends if p == d]
            inn = [c for (p, _, c) in exs[d].recvs if p == s]
            assert out == inn


def test_owned_buckets_match_owner():
    for world in (1, 2, 3, 7, 8):
        for k in (8, 9, 256, 1000):
            if k < world:
                continue
            seen = []
            for r in range(world):
                b0, b1 = sharded.owned_buckets(k, world, r)
                assert all(sharded.bucket_owner(b, k, world) == r for b in range(b0, b1))
                seen += list(range(b0, b1))
            assert seen == list(range(k))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, L, seed, q):
    import torch.distributed as dist

    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = np.arange(n, dtype=np.uint32)
        lo, hi = sharded.slice_bounds(n, world, rank)
        st = sharded.ShardedShuffle(n, 4, k, L, seed, rank, world, device="cpu")
        # level 0 of my slice, from the oracle's draws at the GLOBAL positions (D4)
        ids = oracle.bucket_draws(oracle.problem_key(seed, 0), 0, lo, hi - lo, k)
        grouped = a[lo:hi][np.argsort(ids, kind="stable")]
        st.send[: (hi - lo) * 4].copy_(torch.from_numpy(grouped.view(np.uint8).copy()))
        st.counts.copy_(torch.from_numpy(np.bincount(ids, minlength=k).astype(np.int64)))
        ex = sharded.exchange_plan(sharded.all_gather_counts(st.counts, world), world, k, rank)
        st.exchange(ex, sharded.torch_p2p())
        got = st.result(ex).numpy().view(np.uint32).copy()
        lvl0 = oracle.shuffle(a, k, L, seed, max_levels=1, run_leaves=False)
        q.put((rank, ex.base, ex.m, bool((got == lvl0[ex.base:ex.base + ex.m]).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,world", [(100_003, 256, 2), (50_000, 7, 2), (60_001, 16, 3)])
def test_gloo_ranks_exchange_gives_oracle_level0(n, k, world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, 64, 17, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[3] for r in res] == [True] * world
    at = 0
    for _, base, m, _ in res:  # the owned ranges tile [0, n) in rank order
        assert base == at
        at += m
    assert at == n


def test_capacity_bounds_every_owner():
    """A rank's buffers (capacity) hold its slice and, with a 12-sigma margin, its buckets."""
    rng = np.random.default_rng(3)
    for n, world, k in [(1 << 20, 2, 256), (1 << 22, 8, 1024), (10_007, 3, 7)]:
        cap = sharded.capacity(n, world, k)
        assert cap >= -(-n // world)
        for _ in range(20):
            counts = rng.multinomial(n, [1.0 / k] * k)
            for r in range(world):
                b0, b1 = sharded.owned_buckets(k, world, r)
                assert int(counts[b0:b1].sum()) <= cap


def test_k_smaller_than_world_is_rejected():
    with pytest.raises(ValueError):
        sharded.ShardedShuffle(1000, 4, 2, 16, 1, 0, 4, device="cpu")
