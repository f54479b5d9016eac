"""Sharded single shuffle over G ranks (data sets that
approach memory size, P:9).

ONE problem of N elements -- DESIGN.md D6 with K = seed, bit for bit -- lives
split over G ranks, rank r holding the global positions [lo_r, hi_r) =
[floor(rN/G), floor((r+1)N/G)).  Level 0 (the stable grouping of the whole
array by its level-0 draws) is the only step that crosses ranks;
every later level and every leaf stays inside one level-0 bucket.  So:

1. every rank groups its slice by bucket (``shuf_shard_scatter``: the D4
   draws at the slice's GLOBAL positions, stable, bucket-major) and gets the
   slice's k bucket counts;
2. the counts are all-gathered (G x k int64, one NCCL all-gather);
3. bucket b is owned by rank floor(bG/k) (contiguous bucket ranges); its
   place in the global level-0 output is o_b = sum_{b'<b} tot_b', and inside
   it the pieces come in source-rank order (o_b + sum_{s'<s} c_{s'b}) --
   exactly D6's stable order, because source ranks hold ascending positions.
   The pieces move with one grouped NCCL send/recv batch (an all-to-all-v:
   piece (s, b) is one send on s and one receive on owner(b), issued in
   ascending b on both sides so NCCL pairs them);
4. every owner continues D6 from level 1 on its buckets, in place
   (``shuf_shard_continue``: key K(seed, 0), global positions).

Rank r ends up holding the global output positions [base_r, base_r + m_r)
(base_r = o_{b0(r)}); concatenated over ranks that is D6's output of the
whole problem.  When N <= L, D6 has no level 0 (the array is one leaf): every
rank sends its slice to rank 0, which runs ``shuf_run`` on the whole array.

The data path is the C ABI's kernels plus NCCL; this module is host logic
(exchange layout) and marshalling only.  No CPU fallback: the CUDA entry
points raise when the library or a CUDA tensor is missing.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import paper_2302_03317_b200 as shuf


def slice_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Global positions [lo, hi) of rank's input slice."""
    return (n * rank) // world, (n * (rank + 1)) // world


def owned_buckets(k: int, world: int, rank: int) -> tuple[int, int]:
    """Bucket range [b0, b1) owned by rank: bucket b -> rank floor(b * world / k)."""
    return -(-(rank * k) // world), -(-((rank + 1) * k) // world)


def bucket_owner(b: int, k: int, world: int) -> int:
    return (b * world) // k


@dataclass
class ExchangePlan:
    """Rank r's part of the level-0 all-to-all-v (element units)."""
    rank: int
    base: int                     # global output position of out[0]
    m: int                        # elements this rank owns after the exchange
    child_offsets: list           # owned buckets' boundaries in out, 0 .. m
    sends: list = field(default_factory=list)   # (peer, send offset, length), ascending bucket
    recvs: list = field(default_factory=list)   # (peer, out offset, length), ascending bucket then source
    local: list = field(default_factory=list)   # (send offset, out offset, length): pieces that stay


def exchange_plan(counts, world: int, k: int, rank: int) -> ExchangePlan:
    """counts[s][b] = slice s's count of bucket b (all ranks').  Pure host logic."""
    if len(counts) != world or any(len(c) != k for c in counts):
        raise ValueError("counts must be world x k")
    tot = [sum(int(counts[s][b]) for s in range(world)) for b in range(k)]
    o = [0] * (k + 1)
    for b in range(k):
        o[b + 1] = o[b] + tot[b]
    b0, b1 = owned_buckets(k, world, rank)
    base = o[b0]
    ex = ExchangePlan(rank=rank, base=base, m=o[b1] - o[b0], child_offsets=[o[b] - base for b in range(b0, b1 + 1)])
    # sends: my slice's bucket runs, bucket-major in the send buffer
    src = 0
    mine = [int(c) for c in counts[rank]]
    for b in range(k):
        c = mine[b]
        if c:
            d = bucket_owner(b, k, world)
            if d == rank:
                # where it lands in my own output
                at = o[b] - base + sum(int(counts[s][b]) for s in range(rank))
                ex.local.append((src, at, c))
            else:
                ex.sends.append((d, src, c))
        src += c
    # receives: for each owned bucket, the pieces of every other source in source order
    for b in range(b0, b1):
        at = o[b] - base
        for s in range(world):
            c = int(counts[s][b])
            if c and s != rank:
                ex.recvs.append((s, at, c))
            at += c
    return ex


def _merge_local(pieces):
    """Adjacent local pieces contiguous on both sides become one copy."""
    out = []
    for (src, at, c) in pieces:
        if out and out[-1][0] + out[-1][2] == src and out[-1][1] + out[-1][2] == at:
            out[-1] = (out[-1][0], out[-1][1], out[-1][2] + c)
        else:
            out.append((src, at, c))
    return out


def capacity(n: int, world: int, k: int) -> int:
    """Elements a rank's buffers hold: its slice, or its owned buckets (a
    Binomial(n, (b1-b0)/k) total) with a 12-sigma margin."""
    sl = -(-n // world)
    frac = max(owned_buckets(k, world, r)[1] - owned_buckets(k, world, r)[0] for r in range(world)) / k
    own = n * frac + 12.0 * math.sqrt(n * frac * (1.0 - frac) + 1.0) + 64
    return max(sl, int(own))


def _bytes(t):
    """Flat uint8 view of a contiguous tensor."""
    import torch
    return t.reshape(-1).view(torch.uint8)


class ShardedShuffle:
    """Rank `rank`'s state for sharded shuffles of N elements of eb bytes
    (buffers and scratch allocated once; a step allocates nothing on the GPU
    except the tiny offsets/counts transfers)."""

    def __init__(self, n: int, elem_bytes: int, k: int, L: int, seed: int, rank: int, world: int, device=None):
        import torch
        if elem_bytes not in (4, 8, 16):
            raise ValueError("sharded shuffle: elem_bytes must be 4, 8 or 16")
        if k < world:
            raise ValueError("sharded shuffle needs k >= world (every rank owns a bucket range)")
        self.n, self.eb, self.k, self.L, self.seed = n, elem_bytes, k, L, seed
        self.rank, self.world = rank, world
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lo, self.hi = slice_bounds(n, world, rank)
        self.cap = capacity(n, world, k)
        self.degenerate = n <= L
        pn = n if (self.degenerate and rank == 0) else self.cap
        self.plan = shuf.shuf_plan(max(pn, 1), elem_bytes, k, L, seed)
        sb = shuf.shuf_scratch_bytes(self.plan) if self.degenerate else shuf.shuf_scratch_bytes_shard(self.plan)
        self.scratch = torch.empty(max(sb, 16), dtype=torch.uint8, device=self.device)
        self.out = torch.empty(max(self.cap, n if self.degenerate else 0) * elem_bytes, dtype=torch.uint8,
                               device=self.device)
        # one rank: every piece stays and lands where the scatter put it (no copy)
        self.send = self.out if world == 1 else torch.empty_like(self.out)
        self.counts = torch.zeros(k, dtype=torch.int64, device=self.device)

    # -- step 1: level 0 of my slice ------------------------------------
    def scatter(self, x_local, stream=None):
        m = self.hi - self.lo
        if _bytes(x_local).numel() != m * self.eb:
            raise ValueError(f"rank {self.rank}: slice holds {_bytes(x_local).numel()} bytes, expected {m * self.eb}")
        if self.degenerate:
            self.send[: m * self.eb].copy_(_bytes(x_local))
            return
        shuf.shuf_shard_scatter(self.plan, _bytes(x_local), m, self.lo, self.send, self.counts, self.scratch, stream)

    # -- step 3: the piece moves ----------------------------------------
    def exchange(self, ex: ExchangePlan, p2p):
        """p2p(ops) runs a batch of ("send"|"recv", peer, uint8 tensor view)."""
        eb, ops = self.eb, []
        for (src, at, c) in _merge_local(ex.local):
            if src != at or self.send.data_ptr() != self.out.data_ptr():
                self.out[at * eb:(at + c) * eb].copy_(self.send[src * eb:(src + c) * eb])
        for (d, src, c) in ex.sends:
            ops.append(("send", d, self.send[src * eb:(src + c) * eb]))
        for (s, at, c) in ex.recvs:
            ops.append(("recv", s, self.out[at * eb:(at + c) * eb]))
        p2p(ops)

    # -- step 4: D6 from level 1 on my buckets ---------------------------
    def finish(self, ex: ExchangePlan, stream=None):
        import torch
        if self.degenerate:
            if self.rank == 0 and self.n > 1:
                shuf.shuf_run(self.plan, self.out[: self.n * self.eb], self.scratch, stream)
            return
        if ex.m > self.cap:
            raise RuntimeError(f"rank {self.rank}: owns {ex.m} elements > capacity {self.cap}")
        off = torch.tensor(ex.child_offsets, dtype=torch.int64).to(self.device, non_blocking=True)
        shuf.shuf_shard_continue(self.plan, self.out, ex.m, off, ex.base, 1, self.scratch, stream)

    def degenerate_plan(self) -> ExchangePlan:
        """N <= L: every slice goes to rank 0."""
        m = self.hi - self.lo
        if self.rank == 0:
            ex = ExchangePlan(rank=0, base=0, m=self.n, child_offsets=[0, self.n])
            ex.local.append((0, 0, m))
            for s in range(1, self.world):
                lo, hi = slice_bounds(self.n, self.world, s)
                if hi > lo:
                    ex.recvs.append((s, lo, hi - lo))
            return ex
        ex = ExchangePlan(rank=self.rank, base=self.n, m=0, child_offsets=[0, 0])
        if m:
            ex.sends.append((0, 0, m))
        return ex

    def result(self, ex: ExchangePlan):
        """My part of the output: global positions [ex.base, ex.base + ex.m) (uint8 view)."""
        return self.out[: ex.m * self.eb]


def torch_p2p(group=None):
    """A p2p runner over torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist

    def run(ops):
        if not ops:
            return
        pops = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer, group) for kind, peer, t in ops]
        for w in dist.batch_isend_irecv(pops):
            w.wait()
    return run


def all_gather_counts(counts, world: int, group=None):
    """G x k list of ints from every rank's device counts (one all-gather)."""
    import torch
    import torch.distributed as dist
    bufs = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(bufs, counts, group=group)
    return torch.stack(bufs).cpu().tolist()


def sharded_shuffle(x_local, n: int, k: int, L: int, seed: int, elem_bytes: int | None = None, group=None,
                    state: ShardedShuffle | None = None):
    """This rank's part of D6(N = n) over the process group: returns
    (uint8 view of the owned output, base, m).  x_local = global positions
    slice_bounds(n, world, rank) of the input."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    eb = elem_bytes or x_local.element_size()
    st = state or ShardedShuffle(n, eb, k, L, seed, rank, world, x_local.device)
    st.scatter(x_local)
    if st.degenerate:
        ex = st.degenerate_plan()
    else:
        ex = exchange_plan(all_gather_counts(st.counts, world, group), world, k, rank)
    st.exchange(ex, torch_p2p(group))
    st.finish(ex)
    return st.result(ex), ex.base, ex.m


def simulate_sharded(x, n: int, world: int, k: int, L: int, seed: int, elem_bytes: int | None = None, states=None):
    """All `world` ranks of a sharded shuffle run one after another in THIS
    process on one device (tests, bench): the same kernels and exchange
    layout, the piece moves done as device copies.  Returns the full output
    (uint8) and the per-rank (base, m)."""
    import torch
    eb = elem_bytes or x.element_size()
    xb = _bytes(x)
    sts = states or [ShardedShuffle(n, eb, k, L, seed, r, world, x.device) for r in range(world)]
    for r, st in enumerate(sts):
        xs = xb[st.lo * eb: st.hi * eb]
        if xs.numel() and xs.data_ptr() % 16:  # a real rank's slice is its own allocation
            xs = xs.clone()
        st.scatter(xs)
    if sts[0].degenerate:
        exs = [st.degenerate_plan() for st in sts]
    else:
        counts = torch.stack([st.counts for st in sts]).cpu().tolist()
        exs = [exchange_plan(counts, world, k, r) for r in range(world)]
    # piece moves: every send is matched with the receive of the same (source, dest) pair in order
    for r, (st, ex) in enumerate(zip(sts, exs)):
        for (src, at, c) in _merge_local(ex.local):
            if src != at or st.send.data_ptr() != st.out.data_ptr():
                st.out[at * eb:(at + c) * eb].copy_(st.send[src * eb:(src + c) * eb])
    queues = {}
    for r, (st, ex) in enumerate(zip(sts, exs)):
        for (d, src, c) in ex.sends:
            queues.setdefault((r, d), []).append(st.send[src * eb:(src + c) * eb])
    for r, (st, ex) in enumerate(zip(sts, exs)):
        for (s, at, c) in ex.recvs:
            piece = queues[(s, r)].pop(0)
            if piece.numel() != c * eb:
                raise RuntimeError("exchange layout mismatch between sender and receiver")
            st.out[at * eb:(at + c) * eb].copy_(piece)
    if any(queues.values()):
        raise RuntimeError("unmatched sends in the exchange layout")
    for st, ex in zip(sts, exs):
        st.finish(ex)
    out = torch.empty(n * eb, dtype=torch.uint8, device=x.device)
    for st, ex in zip(sts, exs):
        out[ex.base * eb:(ex.base + ex.m) * eb].copy_(st.result(ex))
    return out, [(ex.base, ex.m) for ex in exs]
