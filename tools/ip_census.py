"""Diagnostic: destination histograms of elements 0 and n-1 over R seeds,
in-place mode vs stable mode (python tools/ip_census.py n R seed0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from scipy import stats  # noqa: E402

from tests.gpu_util import gpu_shuffle  # noqa: E402
from tests.test_gpu_inplace import gpu_inplace  # noqa: E402

n, R, s0 = (int(v) for v in sys.argv[1:4])
a = np.arange(n, dtype=np.uint32)
for name, fn in (("inplace", lambda s: gpu_inplace(a, 2, 1, s)[0]), ("stable", lambda s: gpu_shuffle(a, 2, 1, s))):
    h0 = np.zeros(n, np.int64)
    h1 = np.zeros(n, np.int64)
    for r in range(R):
        got = fn(s0 + r)
        h0[np.flatnonzero(got == 0)[0]] += 1
        h1[np.flatnonzero(got == n - 1)[0]] += 1
    for lab, h in (("first", h0), ("last", h1)):
        hb = h.reshape(-1, 10).sum(1)
        print(name, lab, "p=%.4g" % stats.chisquare(hb).pvalue, "p(all)=%.4g" % stats.chisquare(h).pvalue)
