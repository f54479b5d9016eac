#!/usr/bin/env python
"""Benchmark of the deterministic ScatterShuffle hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hot|c1|c2|c3|c5]
    python bench.py --impl reference ...     # the CPU oracle on a bounded sample

One step = one whole shuffle (every scatter level in HBM and in shared memory
plus the Fisher-Yates leaves) of the workload, resident in HBM, re-shuffling
the previous step's output in place (same cost).  Rank 0 prints
one JSON line.  Under torchrun (N > 1) every rank shuffles its own independent
problem (seed + rank) -- replicas only, weak scaling -- and the
time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "elements shuffled/s and effective HBM GB/s vs 8 TB/s peak, n=2^30 u32"
SPEC_HBM_GBPS = 8000.0
DTYPE = {4: "u32", 8: "u64", 16: "16B-record"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) every ~5 ms on a thread."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.ok = [], 0, None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def workload_bytes(w, stats):
    """Q11 effective bytes: 2*eb*(sum_l n_l + n_leafpass) with n_l every element
    scattered at level l (HBM or shared memory) and the leaf pass over n."""
    scattered = sum(stats["scattered_hbm"]) + sum(stats["scattered_smem"])
    return 2 * w.elem_bytes * (scattered + w.n), scattered


def gpu_baselines(x, n: int, ms_ours: float, dev, reps: int = 3) -> dict:
    """Library GPU shuffles of the same resident input, timed the same way
    (CUDA events, after one warm-up): x[randperm(n)] (PyTorch) and the paper's
    SortShuffle (attach a random key, sort by it) as a CUB radix
    sort of random 64-bit keys.  Uniform shuffles, not D6's permutation:
    comparison points only, never the product path."""
    import torch

    def randperm_gather():
        return x.index_select(0, torch.randperm(n, device=dev))

    def sort_shuffle():
        keys = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), dtype=torch.int64, device=dev)
        return x.index_select(0, torch.sort(keys).indices)

    out = {}
    for name, fn in (("torch_randperm_gather", randperm_gather), ("sort_shuffle_u64_keys", sort_shuffle)):
        try:
            fn()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / reps
            out[name] = {"ms": round(ms, 3), "value": n / (ms / 1e3), "unit": "elements/s",
                         "ours_speedup": round(ms / ms_ours, 2)}
        except RuntimeError as ex:  # out of memory on huge workloads
            out[name] = {"unavailable": str(ex).splitlines()[0][:120]}
        torch.cuda.empty_cache()
    return out


# ---- multi-rank host logic (replicas only); tested with gloo on CPU
def rank_seed(seed: int, rank: int) -> int:
    """Every rank shuffles its own independent problem."""
    return seed + rank


def max_over_ranks(value: float, world: int, device=None) -> float:
    """The job's time is the slowest rank's (all-reduce MAX; nccl on GPU, gloo on CPU)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(n: int, world: int, ms_per_step: float) -> float:
    """Whole-job throughput: elements of all ranks per second of the slowest rank."""
    return n * world / (ms_per_step / 1e3)


def run_reference(args, rank):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    if rank != 0:
        return
    import oracle
    w = synth.WORKLOADS[args.workload]
    n_s = args.ref_sample
    a = synth.make_input_np(w, n=n_s)
    for _ in range(args.warmup):
        oracle.shuffle(a, w.k, w.L, w.seed)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.shuffle(a, w.k, w.L, w.seed)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    v = n_s / dt
    sample = f"{n_s} of the workload's elements ({w.note}, k={w.k}, L={w.L}, seed={w.seed}), one shuffle per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[w.elem_bytes], "data": "synthetic",
            "config": {"workload": args.workload, "n": w.n, "elem_bytes": w.elem_bytes, "k": w.k, "L": w.L,
                       "seed": w.seed},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_sharded(args, w, rank, world, local, dev):
    """--mode sharded (NEXT-3): ONE problem of N = world * n
    elements (the workload's shape per rank, weak scaling), rank r holding
    global positions [rN/world, (r+1)N/world); a step = level-0 scatter of
    the slice, count all-gather, the all-to-all-v of the bucket pieces (NCCL
    grouped send/recv), D6 from level 1 on the owned buckets.  Same input
    slice every step (the scatter reads it, the output goes elsewhere)."""
    import torch
    from paper_2302_03317_b200 import sharded
    import paper_2302_03317_b200 as shuf
    if w.kind == "segmented":
        raise SystemExit("--mode sharded: single-shuffle workloads only")
    N = w.n * world
    st = sharded.ShardedShuffle(N, w.elem_bytes, w.k, w.L, w.seed, rank, world, dev)
    m = st.hi - st.lo
    if w.elem_bytes == 4:
        x = torch.arange(st.lo, st.hi, dtype=torch.int64, device=dev).to(torch.int32)
    else:
        x = synth.make_input_torch(synth.Workload(w.name, m, w.elem_bytes, w.k, w.L, w.seed, w.kind,
                                                  w.num_segments, w.note), dev)
    stream = torch.cuda.current_stream(dev)
    p2p = sharded.torch_p2p()
    info = {}

    def step():
        st.scatter(x, stream)
        if st.degenerate:
            ex = st.degenerate_plan()
        elif world > 1:
            ex = sharded.exchange_plan(sharded.all_gather_counts(st.counts, world), world, w.k, rank)
        else:
            ex = sharded.exchange_plan([st.counts.cpu().tolist()], 1, w.k, 0)
        launches = shuf.shuf_last_launch_count(st.plan)
        st.exchange(ex, p2p)
        st.finish(ex, stream)
        info.update(m=ex.m, base=ex.base, pieces=len(ex.sends) + len(ex.recvs),
                    launches=launches + shuf.shuf_last_launch_count(st.plan))

    for _ in range(max(3, args.warmup)):
        step()
    err = shuf.shuf_last_device_error(st.plan, stream)
    if err:
        raise SystemExit(f"device error {err}")

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    value = N / (ms / 1e3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE[w.elem_bytes], "data": "synthetic",
            "config": {"workload": f"{args.workload} x{world} as ONE sharded problem: N={N}, k={w.k}, L={w.L}, "
                                   f"seed={w.seed}", "n": N, "elem_bytes": w.elem_bytes, "k": w.k, "L": w.L,
                       "seed": w.seed, "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"sharded x{world} (level-0 all-to-all-v over NCCL)", "mode": "sharded",
                       "rank0_owned": info.get("m"), "rank0_p2p_pieces": info.get("pieces")},
            "e2e": None, "roofline": None,
            "cpu_baseline": None if args.no_cpu_baseline else cpu_baseline(w, min(args.cpu_sample, w.n)),
            "gpu_launches": info.get("launches", 0) * args.steps, "clocks": clk.summary(), "device": device_facts(dev),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(w, n_s, mode="stable"):
    """The oracle as it stands on a bounded prefix of the workload: D6 (oracle.shuffle), or
    D10 (oracle.ipsc_shuffle) for --mode ipsc."""
    import oracle
    a = synth.make_input_np(w, n=n_s)
    fn, what = (oracle.ipsc_shuffle, "IpSc (D10)") if mode == "ipsc" else (oracle.shuffle, "D6")
    t0 = time.perf_counter()
    fn(a, w.k, w.L, w.seed)
    dt = time.perf_counter() - t0
    return {"value": n_s / dt, "unit": "elements/s", "cores": 1, "kind": "oracle",
            "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "sample": f"one oracle {what} shuffle of the first {n_s} elements of the workload "
                      f"({w.note}, k={w.k}, L={w.L}, seed={w.seed}); {dt:.1f} s on 1 host core"}


def device_facts(dev) -> dict:
    import torch
    pr = torch.cuda.get_device_properties(dev)
    return {"name": pr.name, "sms": pr.multi_processor_count, "hbm_bytes": pr.total_memory,
            "l2_bytes": getattr(pr, "L2_cache_size", None), "cc": f"{pr.major}.{pr.minor}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hot", choices=["hot", "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="stable", choices=["stable", "inplace", "ipsc", "sharded"],
                    help="inplace: shuf_run_inplace (SURVEY 8(a) a10; aux memory instead of the ping-pong buffer); "
                         "ipsc: shuf_run_ipsc (NEXT-2, the paper's In-Place ScatterShuffle, D10); "
                         "sharded: ONE problem of N x n elements split over the N ranks (NEXT-3, one level-0 "
                         "all-to-all-v over NCCL)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 25)
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--e2e-buffers", type=int, default=2,
                    help="device buffers rotating through the e2e pipeline (2, 3: 105 ms; 4: 119 ms on HOT, r03x)")
    ap.add_argument("--no-gpu-baselines", action="store_true",
                    help="skip the library GPU shuffles timed beside ours (SURVEY 8(f) NEXT-4)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import paper_2302_03317_b200 as shuf

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = synth.WORKLOADS[args.workload]
    if args.mode == "sharded":
        return run_sharded(args, w, rank, world, local, dev)
    seed = rank_seed(w.seed, rank)
    if w.kind == "segmented":
        lens = synth.c5_lengths(w.num_segments, w.seed)
        off_np = synth.segment_offsets(lens)
        n = int(off_np[-1])
        w = synth.Workload(w.name, n, w.elem_bytes, w.k, w.L, w.seed, w.kind, w.num_segments, w.note)
        d_off = torch.from_numpy(off_np.view(np.int64)).to(dev)
        x = synth.make_input_torch(w, dev, offsets=off_np)
    else:
        d_off = None
        x = synth.make_input_torch(w, dev)
    plan = shuf.shuf_plan(w.n, w.elem_bytes, w.k, w.L, seed)
    inplace = args.mode in ("inplace", "ipsc")
    ipsc = args.mode == "ipsc"
    if inplace and d_off is not None:
        raise SystemExit(f"--mode {args.mode}: single-shuffle workloads only")
    if inplace:
        ab = shuf.shuf_aux_bytes_ipsc(plan) if ipsc else shuf.shuf_aux_bytes_inplace(plan)
        scratch = torch.empty(max(16, ab), dtype=torch.uint8, device=dev)
    else:
        scratch = torch.empty(plan.scratch_bytes if d_off is None else plan.scratch_bytes_segmented(d_off.numel() - 1),
                              dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if ipsc:
            shuf.shuf_run_ipsc(plan, x, scratch, stream)
        elif inplace:
            shuf.shuf_run_inplace(plan, x, scratch, stream)
        elif d_off is None:
            shuf.shuf_run(plan, x, scratch, stream)
        else:
            shuf.shuf_segmented(plan, x, d_off, scratch, stream)

    for _ in range(max(3, args.warmup)):
        step()
    err = shuf.shuf_last_device_error(plan, stream)
    if err:
        raise SystemExit(f"device error {err}")
    stats = shuf.shuf_last_run_stats(plan, stream)
    launches_per_step = shuf.shuf_last_launch_count(plan)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    # ---- timed region: K steps, inputs (4 GiB for hot) >> L2, CUDA events on the launching stream
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1), world, dev)
    ms = ms_total / args.steps
    value = job_value(w.n, world, ms)
    eff_bytes, scattered = workload_bytes(w, stats)
    eff_gbps = eff_bytes / (ms / 1e3) / 1e9

    # ---- per-kernel breakdown (separate pass; every launch bracketed by events on `stream`)
    if inplace:  # the in-place mode is one launch of a device-driven CUDA graph: no per-kernel split, the step is the unit
        prof = {c: (0.0, 0) for c in shuf.KERNEL_CLASSES}
        prof["scatter"] = (ms, 1)
    else:
        prof = shuf.shuf_profile_run(plan, x, scratch, d_off, stream)
    peaks, peak_src = load_peaks()
    hbm_peak = float(peaks["hbm_gbs"])
    eb = w.elem_bytes
    kbytes = {"scatter": 2 * eb * sum(stats["scattered_hbm"]), "finish": 2 * eb * stats["finished"],
              "leaf": 2 * eb * stats.get("leafed", 0)}
    kernels = {}
    for name, (kms, cnt) in prof.items():
        d = {"ms": round(kms, 4), "launches": cnt}
        if name in kbytes and kms > 0:
            d["algorithmic_bytes"] = kbytes[name]
            d["GBps"] = round(kbytes[name] / (kms / 1e3) / 1e9, 1)
        kernels[name] = d
    if inplace:  # whole step against the measured copy bandwidth
        kbytes["scatter"] = eff_bytes
    dom = max(("scatter", "finish", "leaf"), key=lambda c: prof[c][0])
    dms, dcnt = prof[dom]
    if dom == "scatter" and not inplace:  # planned-but-empty trailing levels launch and exit at once: count the real ones
        dcnt = max(1, sum(1 for v in stats["scattered_hbm"] if v > 0))
    achieved = kbytes[dom] / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.workload, {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "peak_source": f"{peak_src} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes_per_launch": kbytes[dom] / max(1, dcnt),
                "avg_launch_ms": dms / max(1, dcnt)}
    if inplace:
        roofline["kernel"] = "whole in-place step (Q11 bytes)"

    # ---- end to end through the C ABI with host buffers (pinned), copies timed
    e2e = None
    e2e_fits = True
    if args.e2e_steps > 0 and not inplace:
        # the e2e pipeline rotates >= 2 device buffers and two pinned host buffers of
        # the workload's size; a workload that leaves no room for them (config 4:
        # 64 GiB data + 64 GiB scratch of 178 GiB) reports no e2e number
        need = (max(2, args.e2e_buffers) - 1) * x.numel() * x.element_size()
        e2e_fits = torch.cuda.mem_get_info(dev)[0] > need + (1 << 30)
    if args.e2e_steps > 0 and not inplace and e2e_fits:
        # every step copies its input in from pinned host memory and its result
        # back out; two device buffers let step i+1's upload and step i-1's
        # download run (full duplex) while step i shuffles
        host_in = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        host_in.copy_(x)
        host_out = torch.empty_like(host_in, pin_memory=True)
        nbytes = x.numel() * x.element_size()
        NB = max(2, args.e2e_buffers)
        xbuf = [x] + [torch.empty_like(x) for _ in range(NB - 1)]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(NB)]
        ev_comp = [torch.cuda.Event() for _ in range(NB)]
        ev_out = [torch.cuda.Event() for _ in range(NB)]
        # the link alone, each direction (context for the e2e number)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s_in):
            g0.record(s_in)
            xbuf[1].copy_(host_in, non_blocking=True)
            g1.record(s_in)
        torch.cuda.synchronize(dev)
        h2d_gbps = nbytes / (g0.elapsed_time(g1) / 1e3) / 1e9
        with torch.cuda.stream(s_out):
            g0.record(s_out)
            host_out.copy_(xbuf[1], non_blocking=True)
            g1.record(s_out)
        torch.cuda.synchronize(dev)
        d2h_gbps = nbytes / (g0.elapsed_time(g1) / 1e3) / 1e9

        def run_on(xd):
            if d_off is None:
                shuf.shuf_run(plan, xd, scratch, stream)
            else:
                shuf.shuf_segmented(plan, xd, d_off, scratch, stream)

        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s_in.wait_event(f0)
        s_out.wait_event(f0)
        for i in range(args.e2e_steps):
            d = i % NB
            with torch.cuda.stream(s_in):
                if i >= NB:
                    s_in.wait_event(ev_out[d])  # step i-NB's download has read buffer d
                xbuf[d].copy_(host_in, non_blocking=True)
                ev_in[d].record(s_in)
            stream.wait_event(ev_in[d])
            run_on(xbuf[d])
            ev_comp[d].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[d])
                host_out.copy_(xbuf[d], non_blocking=True)
                ev_out[d].record(s_out)
        stream.wait_event(ev_out[(args.e2e_steps - 1) % NB])
        f1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / args.e2e_steps, world, dev)
        e2e = {"value": job_value(w.n, world, e2e_ms), "unit": "elements/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "overlap": f"uploads, shuffles and downloads of consecutive steps overlap on three streams, "
                          f"{NB} device buffers",
               "link_alone_GBps": {"h2d": round(h2d_gbps, 1), "d2h": round(d2h_gbps, 1)}}
        del host_in, host_out, xbuf

    cpu = None
    gbase = None
    if rank == 0 and world == 1 and not args.no_gpu_baselines and d_off is None:
        gbase = gpu_baselines(x, w.n, ms, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w if w.kind != "segmented" else synth.WORKLOADS["c1"], min(args.cpu_sample, w.n),
                           "ipsc" if ipsc else "stable")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE[w.elem_bytes], "data": "synthetic",
            "config": {"workload": f"{args.workload}: {w.note}, k={w.k}, L={w.L}, seed={w.seed}", "n": w.n,
                       "elem_bytes": w.elem_bytes, "k": w.k, "L": w.L, "seed": w.seed,
                       "l2": "inputs larger than L2 (no flush)" if w.n * w.elem_bytes > (256 << 20)
                       else "input fits in L2: not an HBM figure",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "mode": args.mode,
                       "aux_bytes": int(scratch.numel()) if inplace else None,
                       "scratch_bytes": None if inplace else int(scratch.numel())},
            "eff_GBps": eff_gbps, "frac_of_8TBps": eff_gbps / SPEC_HBM_GBPS,
            "frac_of_measured_copy": eff_gbps / hbm_peak, "effective_bytes_per_step": eff_bytes,
            "elements_scattered_per_step": scattered, "levels": {"hbm": stats["scattered_hbm"],
                                                                 "smem": stats["scattered_smem"]},
            "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "gpu_baselines": gbase, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(), "device": device_facts(dev),
        }
        if not e2e_fits:
            line["e2e_skipped"] = "the e2e pipeline's extra device buffer does not fit beside data + scratch"
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
