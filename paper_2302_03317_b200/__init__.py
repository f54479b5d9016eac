"""paper_2302_03317_b200 -- B200-native deterministic ScatterShuffle hot path.

Thin ctypes binding over ``libshuf.so`` (C ABI in ``include/shuf.h``).  The
names mirror the C entry points; this module only marshals arguments (torch
tensors -> device pointers, torch streams -> cudaStream_t).  Every step of the
shuffle runs in the library's CUDA kernels; there is no CPU fallback: if the
library is missing or no CUDA device is present, calls raise.

    plan = shuf_plan(n, elem_bytes, k, L, seed)
    scratch = torch.empty(shuf_scratch_bytes(plan), dtype=torch.uint8, device="cuda")
    shuf_run(plan, x, scratch)                  # x: contiguous CUDA tensor, n*elem_bytes bytes
    shuf_segmented(plan, x, d_offsets, scratch)
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "ShufError", "lib", "lib_path", "shuf_plan", "shuf_scratch_bytes", "shuf_run", "shuf_segmented",
    "shuf_debug_run_levels", "shuf_debug_bucket_draws", "shuf_debug_fy_draws", "shuf_last_device_error",
    "shuf_destroy", "shuf_planned_levels", "shuf_last_launch_count", "Plan", "shuffle", "segmented_shuffle",
    "EXPORTED_SYMBOLS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("SHUF_LIB_PATH") or os.path.join(_HERE, "libshuf.so")  # env: experiments only
_lib = None

STATUS = {0: "SHUF_OK", 1: "SHUF_ERR_INVALID_ARG", 2: "SHUF_ERR_UNSUPPORTED", 3: "SHUF_ERR_ALIGNMENT",
          4: "SHUF_ERR_SCRATCH", 5: "SHUF_ERR_DEPTH", 6: "SHUF_ERR_CUDA", 7: "SHUF_ERR_RANK_ORDER",
          8: "SHUF_ERR_INTERNAL"}

# every symbol include/shuf.h declares
EXPORTED_SYMBOLS = [
    "shuf_plan", "shuf_last_status", "shuf_scratch_bytes", "shuf_run", "shuf_segmented", "shuf_debug_run_levels",
    "shuf_debug_bucket_draws", "shuf_debug_fy_draws", "shuf_last_device_error", "shuf_last_cuda_error",
    "shuf_last_launch_count", "shuf_planned_levels", "shuf_destroy", "shuf_status_string", "shuf_profile_run",
    "shuf_last_run_stats", "shuf_rank_mode", "shuf_debug_clocks", "shuf_aux_bytes_inplace", "shuf_run_inplace",
    "shuf_scratch_bytes_shard", "shuf_shard_scatter", "shuf_shard_continue", "shuf_aux_bytes_ipsc", "shuf_run_ipsc",
    "shuf_debug_ipsc_levels",
    "shuf_debug_inplace_levels", "shuf_scratch_bytes_segmented", "shuf_sim_rough_scatter",
]
KERNEL_CLASSES = ["init", "hist", "scan", "plan", "scatter", "finish", "leaf"]


class ShufError(RuntimeError):
    def __init__(self, code: int, what: str, cuda_error: int = 0):
        self.code = code
        msg = f"{what}: {STATUS.get(code, code)}"
        if cuda_error:
            msg += f" (cudaError {cuda_error})"
        super().__init__(msg)


def lib():
    """Load libshuf.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} is missing: run `python -m paper_2302_03317_b200._build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(lib_path)
        u32, u64, vp, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.shuf_plan.argtypes = [u64, u32, u32, u32, u64]
        L.shuf_plan.restype = vp
        L.shuf_last_status.restype = i32
        L.shuf_scratch_bytes.argtypes = [vp, ctypes.POINTER(u64)]
        L.shuf_scratch_bytes.restype = i32
        L.shuf_sim_rough_scatter.argtypes = [u64, u32, u64, u32, vp, vp, vp]
        L.shuf_sim_rough_scatter.restype = i32
        L.shuf_scratch_bytes_segmented.argtypes = [vp, u64, ctypes.POINTER(u64)]
        L.shuf_scratch_bytes_segmented.restype = i32
        L.shuf_run.argtypes = [vp, vp, vp, u64, vp]
        L.shuf_run.restype = i32
        L.shuf_segmented.argtypes = [vp, vp, vp, u64, vp, u64, vp]
        L.shuf_segmented.restype = i32
        L.shuf_debug_run_levels.argtypes = [vp, vp, vp, u64, vp, u32, i32]
        L.shuf_debug_run_levels.restype = i32
        L.shuf_debug_bucket_draws.argtypes = [u64, u32, u64, u64, u32, vp, vp]
        L.shuf_debug_bucket_draws.restype = i32
        L.shuf_debug_fy_draws.argtypes = [u64, vp, vp, u64, vp, vp]
        L.shuf_debug_fy_draws.restype = i32
        L.shuf_last_device_error.argtypes = [vp, vp]
        L.shuf_last_device_error.restype = i32
        L.shuf_last_cuda_error.argtypes = [vp]
        L.shuf_last_cuda_error.restype = i32
        L.shuf_last_launch_count.argtypes = [vp]
        L.shuf_last_launch_count.restype = u64
        L.shuf_planned_levels.argtypes = [vp]
        L.shuf_planned_levels.restype = u32
        L.shuf_destroy.argtypes = [vp]
        L.shuf_profile_run.argtypes = [vp, vp, vp, u64, vp, u64, vp, vp, vp]
        L.shuf_profile_run.restype = i32
        L.shuf_last_run_stats.argtypes = [vp, vp, vp, u32]
        L.shuf_last_run_stats.restype = i32
        L.shuf_debug_clocks.argtypes = [vp, vp, vp, u32]
        L.shuf_debug_clocks.restype = i32
        L.shuf_aux_bytes_inplace.argtypes = [vp, ctypes.POINTER(u64)]
        L.shuf_aux_bytes_inplace.restype = i32
        L.shuf_run_inplace.argtypes = [vp, vp, vp, u64, vp]
        L.shuf_run_inplace.restype = i32
        L.shuf_debug_inplace_levels.argtypes = [vp, vp, vp, u64, vp, u32, i32]
        L.shuf_debug_inplace_levels.restype = i32
        L.shuf_rank_mode.restype = i32
        L.shuf_aux_bytes_ipsc.argtypes = [vp, ctypes.POINTER(u64)]
        L.shuf_aux_bytes_ipsc.restype = i32
        L.shuf_run_ipsc.argtypes = [vp, vp, vp, u64, vp]
        L.shuf_run_ipsc.restype = i32
        L.shuf_debug_ipsc_levels.argtypes = [vp, vp, vp, u64, vp, u32, i32]
        L.shuf_debug_ipsc_levels.restype = i32
        L.shuf_scratch_bytes_shard.argtypes = [vp, ctypes.POINTER(u64)]
        L.shuf_scratch_bytes_shard.restype = i32
        L.shuf_shard_scatter.argtypes = [vp, vp, u64, u64, vp, vp, vp, u64, vp]
        L.shuf_shard_scatter.restype = i32
        L.shuf_shard_continue.argtypes = [vp, vp, u64, vp, u64, u64, u32, vp, u64, vp]
        L.shuf_shard_continue.restype = i32
        L.shuf_status_string.argtypes = [i32]
        L.shuf_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


class Plan:
    """Owns a shuf_plan_t; ``handle`` is the raw pointer."""

    def __init__(self, n: int, elem_bytes: int, k: int, L: int, seed: int):
        self.n, self.elem_bytes, self.k, self.L, self.seed = n, elem_bytes, k, L, seed
        h = lib().shuf_plan(n, elem_bytes, k, L, seed % (1 << 64))
        if not h:
            raise ShufError(lib().shuf_last_status(), "shuf_plan")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.shuf_destroy(h)
            self.handle = None

    @property
    def scratch_bytes(self) -> int:
        return shuf_scratch_bytes(self)

    def scratch_bytes_segmented(self, num_segments: int) -> int:
        return shuf_scratch_bytes_segmented(self, num_segments)

    @property
    def planned_levels(self) -> int:
        return shuf_planned_levels(self)


def _check(code: int, what: str, plan: Plan | None = None):
    if code:
        cu = lib().shuf_last_cuda_error(plan.handle) if plan is not None else 0
        raise ShufError(code, what, cu)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dev_ptr(t, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def shuf_plan(n: int, elem_bytes: int, k: int, L: int, seed: int) -> Plan:
    return Plan(n, elem_bytes, k, L, seed)


def shuf_scratch_bytes(plan: Plan) -> int:
    b = ctypes.c_uint64(0)
    _check(lib().shuf_scratch_bytes(plan.handle, ctypes.byref(b)), "shuf_scratch_bytes", plan)
    return int(b.value)


def shuf_scratch_bytes_segmented(plan: Plan, num_segments: int) -> int:
    b = ctypes.c_uint64(0)
    _check(lib().shuf_scratch_bytes_segmented(plan.handle, num_segments, ctypes.byref(b)),
           "shuf_scratch_bytes_segmented", plan)
    return int(b.value)


def shuf_planned_levels(plan: Plan) -> int:
    return int(lib().shuf_planned_levels(plan.handle))


def shuf_last_launch_count(plan: Plan) -> int:
    return int(lib().shuf_last_launch_count(plan.handle))


def _check_data(plan: Plan, x):
    nbytes = x.numel() * x.element_size()
    if nbytes != plan.n * plan.elem_bytes:
        raise ValueError(f"tensor holds {nbytes} bytes, plan expects n*elem_bytes = {plan.n * plan.elem_bytes}")


def shuf_run(plan: Plan, x, scratch, stream=None):
    """Shuffle x in place (stream-ordered; no host sync)."""
    _check_data(plan, x)
    _check(lib().shuf_run(plan.handle, _dev_ptr(x, "x"), _dev_ptr(scratch, "scratch"),
                          scratch.numel() * scratch.element_size(), _stream(stream)), "shuf_run", plan)


def shuf_segmented(plan: Plan, x, d_offsets, scratch, stream=None):
    """Shuffle each segment x[off[s]:off[s+1]] independently (key K(seed, s))."""
    import torch
    _check_data(plan, x)
    if d_offsets.dtype not in (torch.int64, torch.uint64):
        raise ValueError("offsets must be a 64-bit CUDA tensor")
    _check(lib().shuf_segmented(plan.handle, _dev_ptr(x, "x"), _dev_ptr(d_offsets, "offsets"), d_offsets.numel() - 1,
                                _dev_ptr(scratch, "scratch"), scratch.numel() * scratch.element_size(),
                                _stream(stream)), "shuf_segmented", plan)


def shuf_scratch_bytes_shard(plan: Plan) -> int:
    b = ctypes.c_uint64(0)
    _check(lib().shuf_scratch_bytes_shard(plan.handle, ctypes.byref(b)), "shuf_scratch_bytes_shard", plan)
    return int(b.value)


def _check_slice(plan: Plan, x, m: int, what: str):
    if x.numel() * x.element_size() < m * plan.elem_bytes:
        raise ValueError(f"{what} holds fewer than m = {m} elements")


def shuf_shard_scatter(plan: Plan, x, m: int, pos0: int, out, d_counts, scratch, stream=None):
    """Sharded level 0 (include/shuf.h): x[0..m) at global positions pos0.. grouped
    stably by bucket into out[0..m); d_counts (k int64, device) the slice's counts."""
    import torch
    _check_slice(plan, x, m, "x")
    _check_slice(plan, out, m, "out")
    if d_counts.dtype not in (torch.int64, torch.uint64) or d_counts.numel() < plan.k:
        raise ValueError("d_counts must be a 64-bit CUDA tensor of k entries")
    _check(lib().shuf_shard_scatter(plan.handle, _dev_ptr(x, "x"), m, pos0, _dev_ptr(out, "out"),
                                    _dev_ptr(d_counts, "d_counts"), _dev_ptr(scratch, "scratch"),
                                    scratch.numel() * scratch.element_size(), _stream(stream)),
           "shuf_shard_scatter", plan)


def shuf_shard_continue(plan: Plan, x, m: int, d_offsets, base: int, first_level: int, scratch, stream=None):
    """Sharded continuation (include/shuf.h): x[0..m) = global positions base..,
    segments d_offsets (device, int64) are children at first_level; D6 in place."""
    import torch
    _check_slice(plan, x, m, "x")
    if d_offsets.dtype not in (torch.int64, torch.uint64):
        raise ValueError("offsets must be a 64-bit CUDA tensor")
    _check(lib().shuf_shard_continue(plan.handle, _dev_ptr(x, "x"), m, _dev_ptr(d_offsets, "offsets"),
                                     d_offsets.numel() - 1, base, first_level, _dev_ptr(scratch, "scratch"),
                                     scratch.numel() * scratch.element_size(), _stream(stream)),
           "shuf_shard_continue", plan)


def shuf_aux_bytes_ipsc(plan: Plan) -> int:
    v = ctypes.c_uint64(0)
    _check(lib().shuf_aux_bytes_ipsc(plan.handle, ctypes.byref(v)), "shuf_aux_bytes_ipsc", plan)
    return int(v.value)


def shuf_run_ipsc(plan: Plan, x, aux, stream=None):
    """The paper's In-Place ScatterShuffle (NEXT-2, D10): in place, deterministic
    (D10, bit for bit); synchronises the stream once per level."""
    _check_data(plan, x)
    _check(lib().shuf_run_ipsc(plan.handle, _dev_ptr(x, "x"), _dev_ptr(aux, "aux"), aux.numel() * aux.element_size(),
                               _stream(stream)), "shuf_run_ipsc", plan)


def shuf_debug_ipsc_levels(plan: Plan, x, aux, max_levels: int, run_leaves: bool, stream=None):
    _check_data(plan, x)
    _check(lib().shuf_debug_ipsc_levels(plan.handle, _dev_ptr(x, "x"), _dev_ptr(aux, "aux"),
                                        aux.numel() * aux.element_size(), _stream(stream), max_levels,
                                        1 if run_leaves else 0), "shuf_debug_ipsc_levels", plan)


def shuf_aux_bytes_inplace(plan: Plan) -> int:
    v = ctypes.c_uint64(0)
    _check(lib().shuf_aux_bytes_inplace(plan.handle, ctypes.byref(v)), "shuf_aux_bytes_inplace", plan)
    return int(v.value)


def shuf_run_inplace(plan: Plan, x, aux, stream=None):
    """In-place mode (not reproducible; synchronises the stream once per level)."""
    _check_data(plan, x)
    _check(lib().shuf_run_inplace(plan.handle, _dev_ptr(x, "x"), _dev_ptr(aux, "aux"), aux.numel() * aux.element_size(),
                                  _stream(stream)), "shuf_run_inplace", plan)


def shuf_debug_inplace_levels(plan: Plan, x, aux, max_levels: int, run_leaves: bool, stream=None):
    _check_data(plan, x)
    _check(lib().shuf_debug_inplace_levels(plan.handle, _dev_ptr(x, "x"), _dev_ptr(aux, "aux"),
                                           aux.numel() * aux.element_size(), _stream(stream), max_levels,
                                           1 if run_leaves else 0), "shuf_debug_inplace_levels", plan)


def shuf_debug_run_levels(plan: Plan, x, scratch, max_levels: int, run_leaves: bool, stream=None):
    _check_data(plan, x)
    _check(lib().shuf_debug_run_levels(plan.handle, _dev_ptr(x, "x"), _dev_ptr(scratch, "scratch"),
                                       scratch.numel() * scratch.element_size(), _stream(stream), max_levels,
                                       1 if run_leaves else 0), "shuf_debug_run_levels", plan)


def shuf_debug_bucket_draws(K: int, level: int, p0: int, count: int, k: int, out, stream=None):
    _check(lib().shuf_debug_bucket_draws(K % (1 << 64), level, p0, count, k, _dev_ptr(out, "out"), _stream(stream)),
           "shuf_debug_bucket_draws")


def shuf_debug_fy_draws(K: int, q, i, out, stream=None):
    """D5 partners of steps i of the leaves starting at q (device arrays)."""
    _check(lib().shuf_debug_fy_draws(K % (1 << 64), _dev_ptr(q, "q"), _dev_ptr(i, "i"), q.numel(),
                                     _dev_ptr(out, "out"), _stream(stream)), "shuf_debug_fy_draws")


def shuf_sim_rough_scatter(n: int, k: int, seed: int, runs: int, d_T, d_M, stream=None):
    """Hidden-constant simulation (NEXT-1): per run the RoughScatter
    stop time T and the TwoSweep swap count M into int64 CUDA tensors of runs."""
    _check(lib().shuf_sim_rough_scatter(n, k, seed % (1 << 64), runs, _dev_ptr(d_T, "T"), _dev_ptr(d_M, "M"),
                                        _stream(stream)), "shuf_sim_rough_scatter")


def shuf_last_device_error(plan: Plan, stream=None) -> int:
    return int(lib().shuf_last_device_error(plan.handle, _stream(stream)))


def shuf_profile_run(plan: Plan, x, scratch, d_offsets=None, stream=None):
    """Same work as shuf_run / shuf_segmented with every launch bracketed by CUDA
    events on the stream; synchronises.  Returns {class: (ms, launches)}."""
    _check_data(plan, x)
    ms = (ctypes.c_float * len(KERNEL_CLASSES))()
    cnt = (ctypes.c_uint32 * len(KERNEL_CLASSES))()
    offp = _dev_ptr(d_offsets, "offsets") if d_offsets is not None else None
    nseg = d_offsets.numel() - 1 if d_offsets is not None else 0
    _check(lib().shuf_profile_run(plan.handle, _dev_ptr(x, "x"), offp, nseg, _dev_ptr(scratch, "scratch"),
                                  scratch.numel() * scratch.element_size(), _stream(stream), ms, cnt),
           "shuf_profile_run", plan)
    return {KERNEL_CLASSES[i]: (float(ms[i]), int(cnt[i])) for i in range(len(KERNEL_CLASSES))}


def shuf_last_run_stats(plan: Plan, stream=None) -> dict:
    """Device counters of the last run (synchronises): per-level elements
    scattered in HBM / shared memory, elements finished, elements in FY leaves."""
    buf = (ctypes.c_uint64 * 515)()
    _check(lib().shuf_last_run_stats(plan.handle, _stream(stream), buf, 515), "shuf_last_run_stats", plan)
    hbm = [int(buf[2 + 2 * l]) for l in range(256)]
    sm = [int(buf[3 + 2 * l]) for l in range(256)]
    top = max([l + 1 for l in range(256) if hbm[l] or sm[l]] or [0])
    return {"finished": int(buf[0]), "fy_elems": int(buf[1]), "leafed": int(buf[514]),
            "scattered_hbm": hbm[:top], "scattered_smem": sm[:top]}


def shuf_debug_clocks(plan: Plan, stream=None) -> list:
    """Phase clocks of CTA 0 of the fast finish in the last run (6 per item)."""
    buf = (ctypes.c_longlong * 512)()
    _check(lib().shuf_debug_clocks(plan.handle, _stream(stream), buf, 512), "shuf_debug_clocks", plan)
    return [int(buf[i]) for i in range(512)]


def shuf_destroy(plan: Plan):
    plan.__del__()


# ---------------------------------------------------------- convenience ---
def _scratch_for(plan: Plan, device):
    import torch
    return torch.empty(max(1, plan.scratch_bytes), dtype=torch.uint8, device=device)


def shuffle(x, k: int, L: int, seed: int, elem_bytes: int | None = None, scratch=None, stream=None):
    """Shuffle the rows of a contiguous CUDA tensor in place and return it.
    elem_bytes defaults to the row size in bytes (4, 8 or 16)."""
    n = x.shape[0] if x.dim() else 1
    eb = elem_bytes or (x.numel() * x.element_size() // max(1, n))
    plan = shuf_plan(n, eb, k, L, seed)
    shuf_run(plan, x, scratch if scratch is not None else _scratch_for(plan, x.device), stream)
    err = shuf_last_device_error(plan, stream)
    if err:
        raise ShufError(err, "shuf_run (device)")
    return x


def inplace_shuffle(x, k: int, L: int, seed: int, elem_bytes: int | None = None, aux=None, stream=None):
    """In-place mode: shuffle the rows of x with an auxiliary buffer of a few
    percent of x (shuf_aux_bytes_inplace) instead of a full copy."""
    import torch
    n = x.shape[0] if x.dim() else 1
    eb = elem_bytes or (x.numel() * x.element_size() // max(1, n))
    plan = shuf_plan(n, eb, k, L, seed)
    if aux is None:
        aux = torch.empty(max(1, shuf_aux_bytes_inplace(plan)), dtype=torch.uint8, device=x.device)
    shuf_run_inplace(plan, x, aux, stream)
    err = shuf_last_device_error(plan, stream)
    if err:
        raise ShufError(err, "shuf_run_inplace (device)")
    return x


def ipsc_shuffle(x, k: int, L: int, seed: int, elem_bytes: int | None = None, aux=None, stream=None,
                 max_levels: int | None = None, run_leaves: bool = True):
    """The paper's In-Place ScatterShuffle (NEXT-2, D10) of the rows
    of x, in place, with O(k * subtasks) words of aux (shuf_aux_bytes_ipsc)."""
    import torch
    n = x.shape[0] if x.dim() else 1
    eb = elem_bytes or (x.numel() * x.element_size() // max(1, n))
    plan = shuf_plan(n, eb, k, L, seed)
    if aux is None:
        aux = torch.empty(max(16, shuf_aux_bytes_ipsc(plan)), dtype=torch.uint8, device=x.device)
    if max_levels is None:
        shuf_run_ipsc(plan, x, aux, stream)
    else:
        shuf_debug_ipsc_levels(plan, x, aux, max_levels, run_leaves, stream)
    err = shuf_last_device_error(plan, stream)
    if err:
        raise ShufError(err, "shuf_run_ipsc (device)")
    return x


def segmented_shuffle(x, offsets, k: int, L: int, seed: int, elem_bytes: int | None = None, stream=None):
    n = x.shape[0]
    eb = elem_bytes or (x.numel() * x.element_size() // max(1, n))
    plan = shuf_plan(n, eb, k, L, seed)
    import torch
    scratch = torch.empty(max(1, shuf_scratch_bytes_segmented(plan, offsets.numel() - 1)), dtype=torch.uint8,
                          device=x.device)
    shuf_segmented(plan, x, offsets, scratch, stream)
    err = shuf_last_device_error(plan, stream)
    if err:
        raise ShufError(err, "shuf_segmented (device)")
    return x
