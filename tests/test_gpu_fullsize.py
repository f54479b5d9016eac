"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (shuf_run / shuf_segmented on the synth workloads):

- whole-array bit-exact comparison on every config: C1, C2 and C5 directly;
  HOT, C3 and config 4 against whole-array oracle runs computed in worker
  processes while the GPU side runs (tests/oracle_digest.py; per-chunk
  digests are compared, so a mismatch names its chunk);
- config 4 through its permutation pi (SURVEY 8(c) "Config-4 check"): keys
  are the input indices, so key[j] = pi(j); payloads must be intact.

Marked gpu and slow (the config-4 oracle takes a few minutes of one host
core and ~40 GB of host RAM)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2302_03317_b200 as shuf  # noqa: E402

DEV = torch.device("cuda", 0)


def run_workload(name):
    w = synth.WORKLOADS[name]
    x = synth.make_input_torch(w, DEV)
    plan = shuf.shuf_plan(w.n, w.elem_bytes, w.k, w.L, w.seed)
    scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device=DEV)
    shuf.shuf_run(plan, x, scratch)
    assert shuf.shuf_last_device_error(plan) == 0
    del scratch
    return w, x


def test_c1_full_bit_exact():
    w, x = run_workload("c1")
    got = x.cpu().numpy().view(np.uint32)
    exp = oracle.shuffle(synth.make_input_np(w), w.k, w.L, w.seed)
    assert (got == exp).all()


def test_c2_full_bit_exact():
    w, x = run_workload("c2")
    got = x.cpu().numpy().view(np.uint32)
    del x
    exp = oracle.shuffle(synth.make_input_np(w), w.k, w.L, w.seed)
    assert (got == exp).all()


def test_c5_full_bit_exact():
    w = synth.WORKLOADS["c5"]
    off = synth.segment_offsets(synth.c5_lengths(w.num_segments, w.seed))
    n = int(off[-1])
    x = synth.make_input_torch(w, DEV, offsets=off)
    d_off = torch.from_numpy(off.view(np.int64)).to(DEV)
    plan = shuf.shuf_plan(n, 4, w.k, w.L, w.seed)
    scratch = torch.empty(plan.scratch_bytes_segmented(d_off.numel() - 1), dtype=torch.uint8, device=DEV)
    shuf.shuf_segmented(plan, x, d_off, scratch)
    assert shuf.shuf_last_device_error(plan) == 0
    got = x.cpu().numpy().view(np.uint32)
    exp = oracle.segmented(synth.make_input_np(w, offsets=off), off, w.k, w.L, w.seed)
    assert (got == exp).all()


@pytest.fixture(scope="module", autouse=True)
def oracle_jobs():
    """The whole-array oracle runs of HOT, C3 and config 4's permutation, one
    host core each, started when the module starts so they overlap the GPU
    work (tests/oracle_digest.py)."""
    import multiprocessing
    from concurrent.futures import ProcessPoolExecutor

    from tests import oracle_digest
    ex = ProcessPoolExecutor(max_workers=4, mp_context=multiprocessing.get_context("spawn"))
    futs = {name: ex.submit(oracle_digest.job, name) for name in ("c4pi", "c3", "hot", "hot_ipsc")}
    yield futs
    procs = list((ex._processes or {}).values())
    ex.shutdown(wait=False, cancel_futures=True)
    for p in procs:  # a failed run must not wait minutes for unused oracle results
        if p.is_alive():
            p.terminate()


def _gpu_digests(t):
    from tests import oracle_digest
    out = []
    for s in range(0, t.shape[0], oracle_digest.CHUNK):
        out.append(oracle_digest.digests(t[s:s + oracle_digest.CHUNK].cpu().numpy())[0])
    return out


def _assert_same(got, exp, what):
    from tests import oracle_digest
    bad = oracle_digest.first_mismatch(got, exp)
    assert bad is None, f"{what}: chunk {bad} (elements [{bad * oracle_digest.CHUNK}, +{oracle_digest.CHUNK})) differs"


def test_hot_full_bit_exact(oracle_jobs):
    """The metric's run (2^30 u32 iota, k=256, L=4096, seed=1: two HBM levels,
    the pipelined finish on ~16 K-element items, ~64-element leaves), whole
    array against the oracle (P:140-142 stable pi, Fig. 1 leaves P:107-110)."""
    w, x = run_workload("hot")
    got = _gpu_digests(x.view(torch.int32))
    del x
    _assert_same(got, oracle_jobs["hot"].result(), "hot")


def test_hot_sharded_two_ranks_full_bit_exact(oracle_jobs):
    """NEXT-3 at the metric's size: HOT as ONE problem split over two ranks
    (run one after another on this GPU, sharded.simulate_sharded: level-0
    scatter of each slice at its global positions, the exchange layout's
    piece moves, D6 from level 1 on each owner's buckets); the concatenated
    output must equal the single-problem oracle run."""
    from paper_2302_03317_b200 import sharded
    w = synth.WORKLOADS["hot"]
    x = synth.make_input_torch(w, DEV)
    out, parts = sharded.simulate_sharded(x, w.n, 2, w.k, w.L, w.seed, elem_bytes=4)
    del x
    assert parts[0][0] == 0 and parts[0][1] + parts[1][1] == w.n
    got = _gpu_digests(out.view(torch.int32))
    del out
    _assert_same(got, oracle_jobs["hot"].result(), "hot sharded x2")


def test_hot_ipsc_full_bit_exact(oracle_jobs):
    """NEXT-2 at the metric's size: HOT through the paper's In-Place
    ScatterShuffle (shuf_run_ipsc: ParRoughScatter's 2^11 subtasks at the
    root, FineScatter, the small-segment kernel at level 2, leaves), whole
    array against the oracle's D10."""
    w = synth.WORKLOADS["hot"]
    x = synth.make_input_torch(w, DEV)
    shuf.ipsc_shuffle(x, w.k, w.L, w.seed, elem_bytes=4)
    got = _gpu_digests(x.view(torch.int32))
    del x
    _assert_same(got, oracle_jobs["hot_ipsc"].result(), "hot ipsc")


def test_c3_full_bit_exact(oracle_jobs):
    """1,000,000,007 SplitMix64(3) u64 values (ragged tails, partial tiles,
    three HBM levels), whole array against the oracle."""
    w, x = run_workload("c3")
    got = _gpu_digests(x.view(torch.int64))
    del x
    _assert_same(got, oracle_jobs["c3"].result(), "c3")


def test_c4_full_bit_exact_via_pi(oracle_jobs):
    """2^32 16-byte records (64 GiB, k=1024: segments longer than 2^32
    elements take the 64-bit run offsets of the scatter at level 0).  pi is
    independent of the element size (D6), so key[j] must equal the
    oracle's pi(j) computed on u32 iota for every j, and every record must
    arrive whole (payload == splitmix64(key))."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    w = synth.WORKLOADS["c4"]
    if free < 2 * w.n * w.elem_bytes + (8 << 30):
        pytest.skip("needs ~137 GB of free device memory")
    w, x = run_workload("c4")
    step = 1 << 28
    keys = []
    for s in range(0, w.n, step):
        key = x[s:s + step, 0]
        assert bool((synth.splitmix64_of_torch(key) == x[s:s + step, 1]).all())
        assert bool((key >= 0).all() and (key < w.n).all())
        keys.append(key.to(torch.int32))  # keys < 2^32: the u32 bits of pi(j)
    del x
    gc.collect()
    torch.cuda.empty_cache()
    pi = torch.cat(keys)
    del keys
    got = _gpu_digests(pi)
    _assert_same(got, oracle_jobs["c4pi"].result(), "c4 pi")


def test_c4_inplace_bijection_payload_and_block_chi2():
    """BASELINE config 4 asks for the in-place mode at full size too (SURVEY
    8(c) Q14): 2^32 16-byte records shuffled with ~1.4 GB of aux instead of a
    64 GiB ping-pong buffer; every key exactly once with its payload, and the
    one-run (source block, destination block) table over a 64 x 64 grid is
    uniform (chi^2, 3969 dof; each cell expects 2^20 records)."""
    from scipy import stats
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    w = synth.WORKLOADS["c4"]
    if free < w.n * w.elem_bytes + (16 << 30):
        pytest.skip("needs ~80 GB of free device memory")
    x = synth.make_input_torch(w, DEV)
    shuf.inplace_shuffle(x, w.k, w.L, w.seed, elem_bytes=w.elem_bytes)
    seen = torch.zeros(w.n, dtype=torch.bool, device=DEV)
    table = torch.zeros(64 * 64, dtype=torch.int64, device=DEV)
    step = 1 << 28
    for s in range(0, w.n, step):
        key = x[s:s + step, 0]
        assert bool((synth.splitmix64_of_torch(key) == x[s:s + step, 1]).all())
        seen[key] = True
        src = (key.to(torch.int64) & 0xFFFFFFFF) * 64 // w.n
        dst = torch.arange(s, s + key.numel(), device=DEV, dtype=torch.int64) * 64 // w.n
        table += torch.bincount(src * 64 + dst, minlength=64 * 64)
    assert bool(seen.all())
    assert stats.chisquare(table.cpu().numpy()).pvalue > 0.001
