"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, bit-exact (integer work: DESIGN.md section 6)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2302_03317_b200 as shuf  # noqa: E402
from tests.gpu_util import gpu_segmented, gpu_shuffle, to_dev, to_host  # noqa: E402


# ------------------------------------------------------------ raw draws --
@pytest.mark.parametrize("k", [2, 3, 7, 64, 256, 1000, 1024, 40000, 65536])
@pytest.mark.parametrize("level,p0", [(0, 0), (1, 12345), (2, 2**33 + 5), (255, 2**40 - 3)])
def test_raw_bucket_draws(k, level, p0):
    K = oracle.problem_key(9, 4)
    count = 5000
    out = torch.empty(count, dtype=torch.int32, device="cuda")
    shuf.shuf_debug_bucket_draws(K, level, p0, count, k, out)
    got = out.cpu().numpy().view(np.uint32)
    exp = oracle.bucket_draws(K, level, p0, count, k)
    assert (got == exp).all()


def test_raw_fy_draws_including_forced_retries():
    K = oracle.problem_key(11, 2)
    rng = np.random.default_rng(5)
    q = np.concatenate([np.zeros(3000), rng.integers(0, 2**50, size=3000), np.full(300, 12345)]).astype(np.uint64)
    i = np.concatenate([np.arange(1, 3001), rng.integers(1, 2**32 - 1, size=2000), rng.integers(1, 65536, size=1000),
                        np.arange(39900, 40200)]).astype(np.uint32)
    out = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
    shuf.shuf_debug_fy_draws(K, to_dev(q), to_dev(i), out)
    got = out.cpu().numpy().view(np.uint32)
    exp = oracle.fy_draws(K, q, i)
    assert (got == exp).all()
    # s = i+1 near 40000 rejects ~39% of the 16-bit lanes; huge s rejects often too
    assert sum(oracle.fy_draw(K, int(a), int(b))[1] > 0 for a, b in zip(q[-300:], i[-300:])) > 60


# ------------------------------------------------------- end to end ------
CASES = [
    # n, k, L, seed, eb -- several tiles, ragged tails, every path
    (2, 2, 1, 1, 4), (3, 4, 2, 2, 4), (1000, 256, 4096, 3, 4),          # root leaf (FY only)
    (5000, 16, 100, 4, 4),                                              # root fused in smem
    (100_003, 256, 4096, 5, 4),                                         # 1 global level + fused
    (1 << 20, 256, 4096, 1, 4),                                         # config 1
    (777_777, 7, 300, 6, 4),                                            # non-power-of-two k
    (300_001, 1000, 50, 7, 4),                                          # k with rejections
    (200_000, 2, 1, 8, 4),                                              # deepest recursion
    (123_457, 64, 2048, 9, 8), (99_991, 1024, 2048, 10, 16),            # element sizes
    (2_500_000, 256, 4096, 12, 16),                                     # 16-byte leaves of ~L: 2-warp leaf CTAs
    (3_000_000, 256, 4096, 11, 4),                                      # 1 HBM level (+1 planned spare), fused
    (1 << 25, 64, 300, 21, 4),                                          # HOT's shape: 2 HBM levels, then the
    (1 << 26, 256, 64, 22, 4),                                          #  pipelined finish, then FY leaves
    (2_000_000, 256, 1000, 12, 8), (1_000_000, 256, 500, 13, 16),       # fused items of 8/16-byte elements
    (1_500_000, 1024, 600, 14, 16),                                     # k = 1024: several leaves per FY thread
]


def make(n, eb, seed=0):
    if eb == 4:
        return np.arange(n, dtype=np.uint32)
    if eb == 8:
        return synth.splitmix64_stream_np(3 + seed, 0, n)
    return synth.make_input_np(synth.WORKLOADS["c4"], n=n)


@pytest.mark.parametrize("n,k,L,seed,eb", CASES)
def test_shuffle_bit_exact(n, k, L, seed, eb):
    a = make(n, eb)
    got = gpu_shuffle(a, k, L, seed)
    exp = oracle.shuffle(a, k, L, seed)
    assert (got == exp).all()


@pytest.mark.parametrize("n,k,L,seed", [(100_003, 256, 300, 5), (2_000_000, 64, 40, 3), (50_000, 2, 5, 2)])
@pytest.mark.parametrize("max_levels", [0, 1, 2, 3])
@pytest.mark.parametrize("run_leaves", [False, True])
def test_level_limited_state_matches(n, k, L, seed, max_levels, run_leaves):
    """Kernel-level parity: stop after levels l < max_levels (in HBM or in
    shared memory alike) and compare the intermediate state."""
    a = np.arange(n, dtype=np.uint32)
    got = gpu_shuffle(a, k, L, seed, max_levels=max_levels, run_leaves=run_leaves)
    exp = oracle.shuffle(a, k, L, seed, max_levels=max_levels, run_leaves=run_leaves)
    assert (got == exp).all()


def test_segmented_bit_exact_with_edge_segments():
    lens = np.array([0, 1, 2, 5, 4095, 4096, 4097, 30_000, 0, 70_000, 3, 250_000, 1, 0])
    off = synth.segment_offsets(lens)
    a = synth.make_input_np(synth.WORKLOADS["c5"], offsets=off)
    got = gpu_segmented(a, off, 64, 4096, 5)
    exp = oracle.segmented(a, off, 64, 4096, 5)
    assert (got == exp).all()


def test_segmented_c5_shape_sample():
    lens = synth.c5_lengths(4096)
    off = synth.segment_offsets(lens)
    a = synth.make_input_np(synth.WORKLOADS["c5"], offsets=off)
    got = gpu_segmented(a, off, 64, 4096, 5)
    exp = oracle.segmented(a, off, 64, 4096, 5)
    assert (got == exp).all()


def test_repeat_runs_identical_and_stream_independent():
    a = np.arange(1_500_000, dtype=np.uint32)
    r1 = gpu_shuffle(a, 256, 4096, 42)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        r2 = gpu_shuffle(a, 256, 4096, 42)
    assert (r1 == r2).all()
    assert (np.sort(r1) == a).all()


def test_interleaved_plans_share_kernels():
    """Plans of different shapes (k, element size, fused size) used in turn
    in one process: the kernels' shared-memory limits are process-wide, so a
    plan set up later must not break an earlier one."""
    a = np.arange(3_000_000, dtype=np.uint32)
    b = synth.splitmix64_stream_np(3, 0, 400_000)
    c = np.arange(300_001, dtype=np.uint32)
    shapes = [(a, 256, 4096, 11), (b, 1000, 50, 7), (c, 2, 1, 8)]
    plans = []
    for arr, k, L, seed in shapes:
        p = shuf.shuf_plan(arr.shape[0], arr.dtype.itemsize, k, L, seed)
        plans.append((p, torch.empty(p.scratch_bytes, dtype=torch.uint8, device="cuda")))
    for rnd in range(2):
        for (arr, k, L, seed), (p, scr) in zip(shapes, plans):
            x = to_dev(arr)
            shuf.shuf_run(p, x, scr)
            assert shuf.shuf_last_device_error(p) == 0
            assert (to_host(x, arr) == oracle.shuffle(arr, k, L, seed)).all(), (k, L, rnd)


def test_documented_match_rank_path_bit_exact():
    """The ranking fallback (__match_any_sync, SHUF_RANK_MODE=match) is chosen
    once per process, so it runs in a subprocess over every path: HBM levels,
    shared-memory levels (narrow and wide draws), deep recursion, leaves."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, oracle, paper_2302_03317_b200 as shuf\n"
        "from tests.gpu_util import gpu_shuffle\n"
        "cases = [(100_003, 256, 4096, 5), (777_777, 7, 300, 6), (200_000, 2, 1, 8), (3_000_000, 256, 4096, 11),\n"
        "         (300_001, 1000, 50, 7)]\n"
        "for n, k, L, seed in cases:\n"
        "    a = np.arange(n, dtype=np.uint32)\n"
        "    assert (gpu_shuffle(a, k, L, seed) == oracle.shuffle(a, k, L, seed)).all(), (n, k, L, seed)\n"
        "assert shuf.lib().shuf_rank_mode() == 0\n"
        "print('ok')\n" % root)
    env = dict(os.environ, SHUF_RANK_MODE="match")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_WIDE_CASES = (
    "import sys; sys.path.insert(0, %r)\n"
    "import numpy as np, oracle, synth\n"
    "from tests.gpu_util import gpu_shuffle, gpu_segmented\n"
    "for n, k, L, seed in [(3_000_000, 256, 4096, 11), (1 << 25, 64, 300, 21), (777_777, 7, 300, 6),\n"
    "                      (300_001, 1000, 50, 7), (200_000, 2, 1, 8)]:\n"
    "    a = np.arange(n, dtype=np.uint32)\n"
    "    assert (gpu_shuffle(a, k, L, seed) == oracle.shuffle(a, k, L, seed)).all(), (n, k, L, seed)\n"
    "b = synth.splitmix64_stream_np(3, 0, 2_000_000)\n"
    "assert (gpu_shuffle(b, 256, 1000, 12) == oracle.shuffle(b, 256, 1000, 12)).all()\n"
    "c = synth.make_input_np(synth.WORKLOADS['c4'], n=1_500_000)\n"
    "assert (gpu_shuffle(c, 1024, 600, 14) == oracle.shuffle(c, 1024, 600, 14)).all()\n"
    "off = np.array([0, 0, 1, 3000, 300000, 309001, 900000], dtype=np.uint64)\n"
    "d = np.arange(int(off[-1]), dtype=np.uint32)\n"
    "assert (gpu_segmented(d, off, 64, 4096, 5) == oracle.segmented(d, off, 64, 4096, 5)).all()\n"
    "print('ok')\n")


def test_wide_run_offsets_bit_exact():
    """The HBM scatter keeps 64-bit run offsets for segments longer than 2^32
    elements (only config 4's level 0 at full size); SHUF_DBG=64 forces that
    branch for every segment so it is compared with the oracle bit for bit
    at small n (every element size, HBM levels, segmented mode)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _WIDE_CASES % root], env=dict(os.environ, SHUF_DBG="64"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_ENV_CASES = (
    "import sys; sys.path.insert(0, %r)\n"
    "import numpy as np, oracle\n"
    "from tests.gpu_util import gpu_shuffle, gpu_segmented\n"
    "cases = [(3_000_000, 256, 4096, 11), (1 << 20, 256, 4096, 1), (300_001, 1000, 50, 7), (5000, 16, 100, 4),\n"
    "         (777_777, 7, 300, 6), (2_000_000, 64, 40, 3), (4000, 256, 4096, 2), (20_000, 256, 16, 3)]\n"
    "for n, k, L, seed in cases:\n"
    "    a = np.arange(n, dtype=np.uint32)\n"
    "    assert (gpu_shuffle(a, k, L, seed) == oracle.shuffle(a, k, L, seed)).all(), (n, k, L, seed)\n"
    "b = np.arange(400_000, dtype=np.uint64) * 3\n"
    "assert (gpu_shuffle(b, 256, 4096, 5) == oracle.shuffle(b, 256, 4096, 5)).all()\n"
    "off = np.array([0, 0, 1, 3000, 3000, 9000, 9001, 60000, 64000], dtype=np.uint64)\n"
    "c = np.arange(int(off[-1]), dtype=np.uint32)\n"
    "assert (gpu_segmented(c, off, 64, 4096, 5) == oracle.segmented(c, off, 64, 4096, 5)).all()\n"
    "import torch, paper_2302_03317_b200 as shuf\n"
    "d = torch.arange(3_000_000, dtype=torch.int32, device='cuda')\n"
    "shuf.inplace_shuffle(d, 256, 4096, 11)\n"
    "assert (torch.sort(d)[0] == torch.arange(3_000_000, dtype=torch.int32, device='cuda')).all()\n"
    "print('ok')\n")


@pytest.mark.parametrize("env", [{"SHUF_FAST_FINISH": "0"}, {"SHUF_FAST_FINISH": "0", "SHUF_RANK_MODE": "match"},
                                 {"SHUF_LEAF": "0"}, {"SHUF_DEFER": "1", "SHUF_FAST_FINISH": "0"},
                                 {"SHUF_DEFER": "1", "SHUF_FAST_FINISH": "0", "SHUF_RANK_MODE": "match"},
                                 {"SHUF_HIST_LANES": "0"}],
                         ids=["general_finish", "general_finish_match", "no_leaf_kernel", "deferred_leaves",
                              "deferred_leaves_match", "hist_one_table"])
def test_alternate_routes_bit_exact(env):
    """Routes chosen per process by environment (the general finish kernel
    instead of kernels_fast.cu's pipelined one; leaves in the finish kernel
    instead of the leaf kernel; leaves of fused items deferred to the leaf
    kernel) must give the same bits as the oracle on every shape."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ENV_CASES % root], env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_INVARIANCE_CASES = (
    "import sys; sys.path.insert(0, %r)\n"
    "import numpy as np, oracle, synth\n"
    "from tests.gpu_util import gpu_shuffle, gpu_segmented\n"
    "for n, k, L, seed in [(3_000_000, 256, 4096, 11), (1 << 23, 64, 300, 21), (777_777, 7, 300, 6),\n"
    "                      (300_001, 1000, 50, 7), (200_000, 2, 1, 8)]:\n"
    "    a = np.arange(n, dtype=np.uint32)\n"
    "    assert (gpu_shuffle(a, k, L, seed) == oracle.shuffle(a, k, L, seed)).all(), (n, k, L, seed)\n"
    "b = synth.splitmix64_stream_np(3, 0, 1_000_003)\n"
    "assert (gpu_shuffle(b, 256, 1000, 12) == oracle.shuffle(b, 256, 1000, 12)).all()\n"
    "off = np.array([0, 0, 1, 3000, 300000, 309001, 900000], dtype=np.uint64)\n"
    "d = np.arange(int(off[-1]), dtype=np.uint32)\n"
    "assert (gpu_segmented(d, off, 64, 4096, 5) == oracle.segmented(d, off, 64, 4096, 5)).all()\n"
    "print('ok')\n")


@pytest.mark.parametrize("env", [{"SHUF_SFUSE": "5000"}, {"SHUF_CHUNK": "8192"}, {"SHUF_CHUNK": "1000000"},
                                 {"SHUF_GRID": "7"}, {"SHUF_GRID": "1", "SHUF_CHUNK": "40000"}],
                         ids=["sfuse5000", "chunk8192", "chunk1M", "grid7", "grid1"])
def test_schedule_invariance_bit_exact(env):
    """The permutation is a function of (n, k, L, seed) only (D6; the paper's
    schedule independence): the fused size, the chunk size and the
    persistent grid size change which kernel does what and in which order, not
    the bits."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _INVARIANCE_CASES % root], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_depth_overflow_is_reported():
    """A child still longer than the fused size after the last planned HBM
    level must surface as SHUF_ERR_DEPTH through shuf_last_device_error
    (include/shuf.h: callers must check it) -- forced here by planning one HBM
    level (SHUF_LEVELS=1) for a problem that needs two."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import numpy as np\n"
            "from tests.gpu_util import gpu_shuffle\n"
            "import paper_2302_03317_b200 as shuf, torch\n"
            "a = np.arange(1 << 23, dtype=np.uint32)\n"
            "x = torch.from_numpy(a.view(np.int32)).cuda()\n"
            "p = shuf.shuf_plan(a.shape[0], 4, 64, 300, 21)\n"
            "assert p.planned_levels == 1\n"
            "s = torch.empty(p.scratch_bytes, dtype=torch.uint8, device='cuda')\n"
            "shuf.shuf_run(p, x, s)\n"
            "print('err', shuf.shuf_last_device_error(p))\n" % root)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SHUF_LEVELS="1"), capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "err 5" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n,k,L,seed,eb", [(4_000_037, 256, 2048, 41, 8), (3_900_001, 256, 2048, 42, 8),
                                           (5_000_011, 256, 4096, 43, 4)])
def test_stream_finish_bit_exact(n, k, L, seed, eb, monkeypatch):
    """Children between the fused size and the single-buffer size (config-3 shape: ~15 K u64 children)
    finish in k_finish_stream, reading the level's output straight into shared memory; with
    SHUF_STREAM=0 they take another HBM level instead -- both equal the oracle."""
    rng = np.random.default_rng(seed)
    a = np.arange(n, dtype=np.uint32) if eb == 4 else rng.integers(0, 2**63, size=n, dtype=np.uint64)
    exp = oracle.shuffle(a, k, L, seed)
    assert (gpu_shuffle(a, k, L, seed) == exp).all()
    monkeypatch.setenv("SHUF_STREAM", "0")
    assert (gpu_shuffle(a, k, L, seed) == exp).all()


@pytest.mark.parametrize("n,k,L,seed", [(4_200_003, 64, 4096, 51), (600_001, 16, 4096, 52), (9_000_017, 64, 4096, 53)])
def test_leaf_two_pass_slots_bit_exact(n, k, L, seed, monkeypatch):
    """Long leaves expected well below L (config-2 shape: ~L/2) run a first leaf pass with small
    slots and a second pass with full slots for the longer ones.  SHUF_LEAF_SIGMA=0 puts the
    cut at the expected length (about half of the leaves in each pass), -1 is the single pass;
    all equal the oracle (Fig. 1 leaves)."""
    a = np.arange(n, dtype=np.uint32)
    exp = oracle.shuffle(a, k, L, seed)
    assert (gpu_shuffle(a, k, L, seed) == exp).all()
    for sigma in ("0", "-1", "3"):
        monkeypatch.setenv("SHUF_LEAF_SIGMA", sigma)
        assert (gpu_shuffle(a, k, L, seed) == exp).all(), sigma


def test_segmented_long_leaves_bit_exact(monkeypatch):
    """Segmented mode with thousands of long segments (one per warp in the leaf kernel): lengths
    across (0, L], the values around L/2, 3L/4 and L, 0, 1 and L + 1 (D7); SHUF_LEAF_SIGMA=-1
    (no small-slot leaf pass anywhere) gives the same bits."""
    rng = np.random.default_rng(77)
    lens = rng.integers(300, 4097, size=3000).astype(np.int64)
    lens[:12] = [0, 1, 2, 2047, 2048, 2049, 3071, 3072, 3073, 4095, 4096, 4097]
    off = synth.segment_offsets(lens)
    a = np.arange(int(off[-1]), dtype=np.uint32)
    exp = oracle.segmented(a, off, 64, 4096, 9)
    assert (gpu_segmented(a, off, 64, 4096, 9) == exp).all()
    monkeypatch.setenv("SHUF_LEAF_SIGMA", "-1")
    assert (gpu_segmented(a, off, 64, 4096, 9) == exp).all()
