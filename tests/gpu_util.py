"""Helpers for the -m gpu parity tests: move numpy arrays through the C-ABI
library (paper_2302_03317_b200) and back, bit for bit."""
import numpy as np
import torch

import paper_2302_03317_b200 as shuf

_SIGNED = {np.dtype(np.uint8): np.int8, np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64}


def to_dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    sd = _SIGNED.get(a.dtype, a.dtype)
    return torch.from_numpy(a.view(sd)).cuda()


def to_host(t: torch.Tensor, like: np.ndarray) -> np.ndarray:
    return t.cpu().numpy().view(like.dtype).reshape(like.shape)


def elem_bytes(a: np.ndarray) -> int:
    return a.strides[0] if a.ndim > 1 else a.dtype.itemsize


def gpu_shuffle(a: np.ndarray, k: int, L: int, seed: int, max_levels=None, run_leaves=True, check_err=True):
    x = to_dev(a)
    n = a.shape[0]
    plan = shuf.shuf_plan(n, elem_bytes(a), k, L, seed)
    scratch = torch.empty(max(1, plan.scratch_bytes), dtype=torch.uint8, device="cuda")
    if max_levels is None:
        shuf.shuf_run(plan, x, scratch)
    else:
        shuf.shuf_debug_run_levels(plan, x, scratch, max_levels, run_leaves)
    err = shuf.shuf_last_device_error(plan)
    if check_err:
        assert err == 0, (err, shuf.lib().shuf_last_cuda_error(plan.handle))
    return to_host(x, a)


def gpu_segmented(a: np.ndarray, offsets: np.ndarray, k: int, L: int, seed: int):
    x = to_dev(a)
    off = torch.from_numpy(np.asarray(offsets, dtype=np.uint64).view(np.int64)).cuda()
    plan = shuf.shuf_plan(a.shape[0], elem_bytes(a), k, L, seed)
    scratch = torch.empty(max(1, plan.scratch_bytes_segmented(off.numel() - 1)), dtype=torch.uint8, device="cuda")
    shuf.shuf_segmented(plan, x, off, scratch)
    assert shuf.shuf_last_device_error(plan) == 0
    return to_host(x, a)
