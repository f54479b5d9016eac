"""Run one GPU shuffle case through the C ABI and compare with the oracle.
usage: python tools/repro_case.py n k L seed [eb]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from tests.gpu_util import gpu_shuffle  # noqa: E402

n, k, L, seed = (int(x) for x in sys.argv[1:5])
a = np.arange(n, dtype=np.uint32)
got = gpu_shuffle(a, k, L, seed)
exp = oracle.shuffle(a, k, L, seed)
print("match", bool((got == exp).all()))
