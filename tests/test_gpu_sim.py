"""GPU parity of the hidden-constant simulation (NEXT-1, D9,
PAPER.md P:773-788): per run, the RoughScatter stop time T and the TwoSweep
swap count M from the C-ABI kernel equal the oracle's bit for bit (integer
results), for power-of-two and general k, packed-u16 counters (k > 2^15),
ragged n and several tiles per run."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2302_03317_b200 as shuf  # noqa: E402


def gpu_sim(n, k, seed, runs):
    T = torch.zeros(runs, dtype=torch.int64, device="cuda")
    M = torch.zeros(runs, dtype=torch.int64, device="cuda")
    shuf.shuf_sim_rough_scatter(n, k, seed, runs, T, M)
    torch.cuda.synchronize()
    return T.cpu().numpy().view(np.uint64), M.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("n,k,seed,runs", [
    (4, 2, 1, 2000), (1000, 3, 2, 300), (100_003, 64, 3, 200), (1 << 20, 256, 4, 64), (300_001, 1000, 5, 64),
    (4_000_037, 40_000, 6, 16), (1 << 22, 65_536, 7, 8), (65_536, 65_536, 8, 16),
])
def test_sim_bit_exact(n, k, seed, runs):
    gT, gM = gpu_sim(n, k, seed, runs)
    eT, eM = oracle.sim_rough_scatter(n, k, seed, runs)
    assert (gT == eT).all()
    assert (gM == eM).all()


def test_sim_domain_errors():
    T = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(shuf.ShufError):
        shuf.shuf_sim_rough_scatter(10, 1, 1, 1, T, T)
    with pytest.raises(shuf.ShufError):
        shuf.shuf_sim_rough_scatter(1 << 40, 65_536, 1, 1, T, T)  # counts would overflow u16
