"""Pins for the oracle's shuffle.  Expected values come
from library routines (numpy's stable argsort), the paper's Fig. 1 loop with a
stub generator, closed forms (multinomial moments), invariants
(bijection), and chi-square goodness of fit against the exact uniform
distribution over permutations ("1 and 2-independence of the output
ranks")."""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
import synth
from tests.ref_numpy import shuffle_np

ALPHA = 1e-3


def perm_index(P: np.ndarray) -> np.ndarray:
    """Lehmer code (factorial number system) of each row of P."""
    P = np.asarray(P, dtype=np.int64)
    r, n = P.shape
    idx = np.zeros(r, dtype=np.int64)
    for i in range(n):
        smaller = (P[:, i + 1:] < P[:, i:i + 1]).sum(axis=1)
        idx = idx * (n - i) + smaller
    return idx


# ------------------------------------------------------------ scatter ----
@pytest.mark.parametrize("n,k,seed", [(10_000, 256, 1), (7_777, 7, 2), (5_000, 1000, 3), (4096 * 3 + 5, 64, 4)])
def test_one_level_equals_stable_argsort(n, k, seed):
    """Level 0 with max_levels=1, no leaves: OUT = IN[argsort(A, stable)] where
    A are the D4 draws (pi chosen stable)."""
    a = np.arange(n, dtype=np.uint32)
    out = oracle.shuffle(a, k, 1, seed, max_levels=1, run_leaves=False)
    A = oracle.bucket_draws(oracle.problem_key(seed, 0), 0, 0, n, k)
    assert (out == a[np.argsort(A, kind="stable")]).all()


def test_two_levels_equal_nested_stable_argsort():
    """Level 1 sorts each child segment (> L) of level 0 by level-1 draws at
    its problem-relative positions; children <= L stay (no leaves run)."""
    n, k, L, seed = 50_000, 16, 700, 9
    K = oracle.problem_key(seed, 0)
    a = np.arange(n, dtype=np.uint32)
    got = oracle.shuffle(a, k, L, seed, max_levels=2, run_leaves=False)
    A0 = oracle.bucket_draws(K, 0, 0, n, k)
    exp = a[np.argsort(A0, kind="stable")]
    cnt = np.bincount(A0, minlength=k)
    start = 0
    for c in cnt:
        if c > L:
            A1 = oracle.bucket_draws(K, 1, start, int(c), k)
            exp[start:start + c] = exp[start:start + c][np.argsort(A1, kind="stable")]
        start += int(c)
    assert (got == exp).all()


# ------------------------------------------------------------ FY ---------
def test_fy_stub_trace_S116():
    """Fig. 1 with gen_index == 0 maps [a,b,c] -> [b,c,a]."""
    out = oracle.fy_with_draws(np.array([10, 11, 12], dtype=np.uint32), [0, 0, 0])
    assert list(out) == [11, 12, 10]
    assert list(oracle.fy_with_draws(np.array([5], dtype=np.uint32), [0])) == [5]


def test_fy_stub_identity_draws():
    """j_i = i for every step leaves the array unchanged (swap with itself)."""
    a = np.arange(9, dtype=np.uint64) * 3
    assert (oracle.fy_with_draws(a, np.arange(9)) == a).all()


@pytest.mark.parametrize("n", [2, 3, 100, 4096])
def test_single_leaf_is_textbook_fisher_yates(n):
    """With L >= n the whole problem is one leaf: Fig. 1 loop (i = n-1..1,
    swap A[i], A[j], j in [0,i]) with the D5 draws."""
    seed = 31 + n
    K = oracle.problem_key(seed, 0)
    a = np.arange(n, dtype=np.uint32)
    got = oracle.shuffle(a, 2, n, seed)
    i = np.arange(n - 1, 0, -1)
    j = oracle.fy_draws(K, 0, i)  # leaf id = its start position 0, step i
    assert (j <= i).all()
    exp = list(range(n))
    for ii, jj in zip(i, j):
        exp[ii], exp[jj] = exp[jj], exp[ii]
    assert list(got) == exp


# ------------------------------------------------------------ census -----
CENSUS = [  # (n, k, L): forcing 0, 1, 2 and many scatter levels
    (3, 2, 1), (4, 4, 1), (5, 2, 1), (5, 2, 3), (5, 256, 1), (5, 2, 5), (6, 3, 2), (8, 2, 2),
]


@pytest.mark.parametrize("n,k,L", CENSUS)
def test_census_all_permutations_uniform(n, k, L):
    """Brute force over n! cells (north star: n<=8, 10^6 seeds, chi-square
    p > 0.001; Bonferroni over the family).  10^6 independent problems
    via D7 (distinct keys K(seed, s))."""
    R = 1_000_000
    data = np.tile(np.arange(n, dtype=np.uint32), R)
    off = np.arange(R + 1, dtype=np.uint64) * n
    out = oracle.segmented(data, off, k, L, 1000 + n).reshape(R, n)
    assert (np.sort(out, axis=1) == np.arange(n)).all()  # bijection per run
    cells = np.bincount(perm_index(out), minlength=math.factorial(n))
    p = stats.chisquare(cells).pvalue
    assert p > ALPHA / len(CENSUS), (n, k, L, p)


def test_rank_1_and_2_independence_n32():
    """P:557 / S:137-138: (element, position) cells uniform at n=32; joint
    positions of elements (0,1) uniform over the 32*31 ordered pairs."""
    n, R = 32, 100_000
    data = np.tile(np.arange(n, dtype=np.uint32), R)
    off = np.arange(R + 1, dtype=np.uint64) * n
    out = oracle.segmented(data, off, 4, 3, 77).reshape(R, n)
    pos = np.argsort(out, axis=1)  # pos[r, e] = output position of element e
    table = np.zeros((n, n), dtype=np.int64)
    for e in range(n):
        table[e] = np.bincount(pos[:, e], minlength=n)
    p1 = stats.chisquare(table.ravel()).pvalue
    pair = pos[:, 0] * n + pos[:, 1]
    cells = np.bincount(pair, minlength=n * n).reshape(n, n)
    assert (np.diag(cells) == 0).all()
    p2 = stats.chisquare(cells[~np.eye(n, dtype=bool)]).pvalue
    assert p1 > ALPHA / 2 and p2 > ALPHA / 2, (p1, p2)


# ------------------------------------------------------- multinomial -----
def test_level0_bucket_sizes_multinomial_moments():
    """bucket sizes follow multinomial(n, 1/k): mean n/k, variance
    n(1/k)(1-1/k), covariance -n/k^2 (within sampling error)."""
    n, k, S = 1 << 16, 256, 400
    C = np.empty((S, k), dtype=np.float64)
    for s in range(S):
        A = oracle.bucket_draws(oracle.problem_key(100 + s, 0), 0, 0, n, k)
        C[s] = np.bincount(A, minlength=k)
    assert (C.sum(axis=1) == n).all()
    mean, var = n / k, n * (1 / k) * (1 - 1 / k)
    se_mean = math.sqrt(var / (S * k))
    assert abs(C.mean() - mean) < 1e-9  # exact: rows sum to n
    # every bucket's mean within 5 standard errors
    assert (np.abs(C.mean(axis=0) - mean) < 5 * math.sqrt(var / S)).all()
    # pooled variance within 5% (S*k = 102400 samples), covariance of adjacent buckets
    v = C.var(axis=0, ddof=1).mean()
    assert abs(v / var - 1) < 0.05, v / var
    cov = np.mean([np.cov(C[:, b], C[:, b + 1])[0, 1] for b in range(0, k - 1, 2)])
    assert abs(cov - (-n / k**2)) < 0.2 * var / math.sqrt(S) * 5, cov
    # one-run chi-square of the k sizes against uniform (255 dof)
    p = stats.chisquare(C[0]).pvalue
    assert p > ALPHA
    del se_mean


# ------------------------------------------------------ invariants -------
@pytest.mark.parametrize("n,k,L,seed", [(0, 4, 4, 1), (1, 4, 4, 1), (2, 2, 1, 5), (100, 2, 1, 3),
                                        (12_345, 7, 50, 8), (70_000, 256, 4096, 1), (33_333, 1024, 20, 2)])
def test_bijection_and_levels(n, k, L, seed):
    a = np.arange(n, dtype=np.uint32)
    out, st = oracle.shuffle(a, k, L, seed, stats=True)
    assert (np.sort(out) == a).all()
    if n > L:
        assert st["scatter_elems"][0] == n
        assert all(x <= n for x in st["scatter_elems"])


def test_permutation_independent_of_element_type_Q9():
    """pi depends on (n, k, L, seed) only: u64 values and 16-B records move as
    the gather of the iota run says."""
    n, k, L, seed = 30_001, 64, 200, 13
    pi = oracle.shuffle(np.arange(n, dtype=np.uint32), k, L, seed).astype(np.int64)
    v = synth.splitmix64_stream_np(3, 0, n)
    assert (oracle.shuffle(v, k, L, seed) == v[pi]).all()
    rec = synth.make_input_np(synth.WORKLOADS["c4"], n=n)
    assert (oracle.shuffle(rec, k, L, seed) == rec[pi]).all()
    b = np.arange(n, dtype=np.uint8)
    assert (oracle.shuffle(b, k, L, seed) == b[pi]).all()


def test_segmented_equals_single_with_folded_key_Q8():
    lens = np.array([0, 1, 5, 4096, 4097, 9000, 2, 0, 3000])
    off = synth.segment_offsets(lens)
    data = synth.make_input_np(synth.WORKLOADS["c5"], offsets=off)
    k, L, seed = 64, 4096, 5
    out = oracle.segmented(data, off, k, L, seed)
    for s in range(len(lens)):
        a, b = int(off[s]), int(off[s + 1])
        single = oracle.shuffle(data[a:b], k, L, oracle.problem_key(seed, s))
        assert (out[a:b] == single).all()
        assert (np.sort(out[a:b]) == np.arange(b - a)).all()


def test_depth_limited_then_leaves_only():
    """max_levels=0 with run_leaves: a root <= L is still finished by FY;
    a root > L is left untouched."""
    a = np.arange(100, dtype=np.uint32)
    assert (oracle.shuffle(a, 4, 50, 1, max_levels=0) == a).all()
    assert not (oracle.shuffle(a, 4, 100, 1, max_levels=0) == a).all()


# ------------------------------------------- second implementation -------
@pytest.mark.parametrize("n,k,L,seed", [(1, 2, 1, 1), (37, 2, 1, 2), (500, 3, 7, 3), (3000, 256, 10, 4),
                                        (9000, 1000, 5, 5), (20_000, 16, 300, 6), (4000, 4, 4000, 7)])
def test_oracle_matches_independent_numpy_derivation(n, k, L, seed):
    a = np.arange(n, dtype=np.uint32)
    got = oracle.shuffle(a, k, L, seed)
    exp = shuffle_np(a, k, L, oracle.problem_key(seed, 0))
    assert (got == exp).all()


@pytest.mark.parametrize("n,k,L,seed", [(1, 2, 1, 1), (2, 2, 1, 1), (37, 2, 1, 2), (5000, 7, 30, 3),
                                        (100_003, 256, 300, 5), (300_001, 1000, 50, 7), (200_000, 2, 1, 8),
                                        (1 << 20, 256, 4096, 1)])
def test_point_queries_equal_full_shuffle(n, k, L, seed):
    """oracle.points (the D6 walk used for sampled checks at full size) resolves
    every queried output position to the same input index as the full D6."""
    pi = oracle.shuffle(np.arange(n, dtype=np.uint64), k, L, seed)
    js = np.arange(n, dtype=np.uint64) if n <= 5000 else np.random.default_rng(seed).integers(0, n, 300).astype(np.uint64)
    assert (oracle.points(n, k, L, seed, js) == pi[js.astype(np.int64)]).all()
