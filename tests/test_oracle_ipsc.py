"""Pins of the oracle's paper-faithful In-Place ScatterShuffle (D10;
SURVEY 8(f) NEXT-2; RoughScatter P:262-265, ParRoughScatter P:479-491,
FineScatter P:357-425).  Checked against what the paper and the mathematics
fix, not against the oracle itself:
  - every run is a bijection, and the permutation does not depend on the
    element size;
  - the n! census of tiny inputs is uniform (chi^2, Bonferroni);
  - the final level-0 bucket sizes are multinomial(n, 1/k) in mean, variance
    and covariance (N^f = N + N' is multinomial);
  - RoughScatter leaves R <= sqrt(2 n k ln k) staged items whp (Lemma 2,
    P:284-296; also after ParRoughScatter's merges, Observation P:493);
  - TwoSweep moves sum_i |D_i| items (Lemma 4) -- checked against the
    prefix sums of the returned final sizes, recomputed here;
  - the destination of a fixed element is uniform (Lemma 1 + Lemma 3).
"""
import math
from collections import Counter

import numpy as np
import pytest
from scipy import stats

import oracle


@pytest.mark.parametrize("n,k,L", [(2, 2, 1), (7, 2, 1), (1000, 4, 16), (65_537, 16, 64), (200_003, 256, 300),
                                   (50_000, 3, 5), (30_000, 1000, 40)])
def test_bijection_and_element_size_independence(n, k, L):
    a = np.arange(n, dtype=np.uint32)
    b = oracle.ipsc_shuffle(a, k, L, 11)
    assert np.array_equal(np.sort(b), a)
    rec = np.zeros((n, 2), dtype=np.uint64)
    rec[:, 0] = np.arange(n)
    rec[:, 1] = np.arange(n) * 7919
    r = oracle.ipsc_shuffle(rec, k, L, 11)
    assert np.array_equal(r[:, 0].astype(np.uint32), b)
    assert np.array_equal(r[:, 1], r[:, 0] * 7919)


@pytest.mark.parametrize("n,k,L", [(4, 2, 1), (5, 2, 1), (5, 3, 1), (6, 2, 2)])
def test_census_uniform(n, k, L):
    seeds = 24 * math.factorial(n)
    cnt = Counter()
    base = np.arange(n, dtype=np.uint32)
    for s in range(seeds):
        cnt[tuple(oracle.ipsc_shuffle(base, k, L, s))] += 1
    assert len(cnt) == math.factorial(n)
    obs = np.array(list(cnt.values()), dtype=float)
    p = stats.chisquare(obs).pvalue
    assert p > 0.001 / 4, p


def test_final_sizes_are_multinomial():
    n, k, runs = 20_000, 16, 400
    assert oracle.ipsc_depth(n, k) == 6  # ParRoughScatter merges on 6 levels
    S = np.zeros((runs, k))
    for r in range(runs):
        _, st, sizes = oracle.ipsc_shuffle(np.arange(n, dtype=np.uint32), k, 64, 1000 + r, max_levels=1,
                                           run_leaves=False, stats=True)
        S[r] = sizes
        assert sizes.sum() == n
    p = 1.0 / k
    mean, var = n * p, n * p * (1 - p)
    # mean of every bucket within 4.5 standard errors; pooled variance within 15 %
    assert np.all(np.abs(S.mean(0) - mean) < 4.5 * math.sqrt(var / runs))
    assert abs(S.var(0, ddof=1).mean() / var - 1) < 0.15
    cov = np.cov(S.T)[np.triu_indices(k, 1)].mean()
    assert abs(cov / (-n * p * p) - 1) < 0.25


def test_lemma2_staged_bound():
    n, k, runs = 1 << 18, 64, 60
    bound = math.sqrt(2 * n * k * math.log(k))
    R = []
    for r in range(runs):
        _, st, _ = oracle.ipsc_shuffle(np.arange(n, dtype=np.uint32), k, 4096, 7 + r, max_levels=1,
                                       run_leaves=False, stats=True)
        R.append(st["staged"])
    R = np.array(R, dtype=float)
    assert (R <= bound).mean() >= 0.9
    assert 0.4 < R.mean() / bound < 1.0


def test_twosweep_moves_sum_of_abs_prefix_deviations():
    for n, k in [(10_007, 8), (65_536, 64), (3000, 3)]:
        _, st, sizes = oracle.ipsc_shuffle(np.arange(n, dtype=np.uint32), k, 16, 3, max_levels=1,
                                           run_leaves=False, stats=True)
        cap = np.array([(i + 1) * n // k - i * n // k for i in range(k)], dtype=np.int64)
        D = np.cumsum(sizes.astype(np.int64) - cap)
        assert st["transfers"] == np.abs(D).sum() == st["dsum"]
        assert st["segments"] == 1


def test_destination_of_an_element_is_uniform():
    n, k, L, runs, bins = 3000, 8, 16, 3000, 20
    h0, hm = np.zeros(bins), np.zeros(bins)
    base = np.arange(n, dtype=np.uint32)
    for r in range(runs):
        b = oracle.ipsc_shuffle(base, k, L, 50_000 + r)
        inv = np.empty(n, dtype=np.int64)
        inv[b] = np.arange(n)
        h0[inv[0] * bins // n] += 1
        hm[inv[n // 2] * bins // n] += 1
    assert stats.chisquare(h0).pvalue > 0.0005
    assert stats.chisquare(hm).pvalue > 0.0005


def test_draw_layout_from_pinned_primitives():
    """D10 draws compose the pinned Philox (cuRAND) and Lemire32 (exhaustive)."""
    K = oracle.problem_key(9, 0)
    for tag, c0, c1, lvl, a, bound in [(7, 0, 1, 0, 0, 256), (8, 12345, 0, 3, 2**40 + 5, 1000), (9, 77, 0, 1, 99, 78)]:
        w = oracle.philox([c0, c1, a & 0xFFFFFFFF, tag | (lvl << 8) | (((a >> 32) & 0xFFFF) << 16)],
                          [K & 0xFFFFFFFF, K >> 32])
        exp = None
        for x in w:
            v = oracle.lemire32(int(x), bound)  # None on rejection
            if v is not None:
                exp = v
                break
        assert oracle.ipsc_draw(K, tag, c0, c1, lvl, a, bound) == exp


def test_depth_rule():
    assert oracle.ipsc_depth(255, 16) == 0
    assert oracle.ipsc_depth(512, 16) == 1
    assert oracle.ipsc_depth(1 << 40, 16) == 11
    assert oracle.ipsc_depth(1 << 30, 256) == 11
    assert oracle.ipsc_depth((1 << 16) * 3, 256) == 1
