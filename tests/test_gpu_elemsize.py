"""Element sizes other than 4, 8 and 16 bytes (the paper's
element-size experiment, Fig. 7): the library shuffles
the index array with the native kernels and moves each element once (the
gather route, kernels_gather.cu).  D6's permutation depends on (n, k, L, seed)
only, so the result must equal the oracle's shuffle of the same rows bit for
bit, whatever the row size."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2302_03317_b200 as shuf  # noqa: E402
from tests.gpu_util import gpu_segmented, gpu_shuffle  # noqa: E402


def rows(n: int, eb: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 256, size=(n, eb), dtype=np.uint8)


@pytest.mark.parametrize("eb", [1, 2, 3, 12, 24, 32, 64, 256])
@pytest.mark.parametrize("n,k,L,seed", [(1000, 256, 4096, 3), (300_001, 256, 4096, 5), (200_000, 7, 100, 6)])
def test_gather_route_bit_exact(eb, n, k, L, seed):
    if eb == 256 and n > 250_000:
        n = 120_001
    a = rows(n, eb, seed + eb)
    got = gpu_shuffle(a, k, L, seed)
    assert (got == oracle.shuffle(a, k, L, seed)).all()


@pytest.mark.parametrize("eb", [1, 32, 64])
def test_gather_route_two_hbm_levels(eb):
    n = 1 << 22
    a = rows(n, eb, 41) if eb > 1 else rows(n, 1, 41)
    got = gpu_shuffle(a, 64, 300, 21)
    assert (got == oracle.shuffle(a, 64, 300, 21)).all()


def test_gather_route_equals_native_permutation():
    # the same (n, k, L, seed) moves 4-byte and 32-byte rows by the same permutation
    n = 500_000
    idx = np.arange(n, dtype=np.uint32)
    perm = gpu_shuffle(idx, 256, 4096, 9)
    a = rows(n, 32, 9)
    assert (gpu_shuffle(a, 256, 4096, 9) == a[perm]).all()


@pytest.mark.parametrize("eb", [2, 32])
def test_gather_route_segmented(eb):
    lens = np.random.default_rng(3).integers(0, 9000, size=300)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    a = rows(int(off[-1]), eb, 7)
    got = gpu_segmented(a, off, 64, 4096, 5)
    assert (got == oracle.segmented(a, off, 64, 4096, 5)).all()


@pytest.mark.parametrize("eb", [1, 64])
def test_gather_route_level_limited(eb):
    a = rows(400_000, eb, 8)
    for lv in (0, 1):
        got = gpu_shuffle(a, 16, 64, 4, max_levels=lv, run_leaves=False)
        assert (got == oracle.shuffle(a, 16, 64, 4, max_levels=lv, run_leaves=False)).all()


def test_gather_route_has_no_inplace_mode():
    plan = shuf.shuf_plan(1000, 32, 16, 64, 1)
    with pytest.raises(shuf.ShufError):
        shuf.shuf_aux_bytes_inplace(plan)
