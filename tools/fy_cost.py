#!/usr/bin/env python
"""Measure the Fisher-Yates share of a run: time the whole shuffle with and
without the leaf pass (shuf_debug_run_levels, run_leaves 1 vs 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
import synth  # noqa: E402

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hot"]
x = synth.make_input_torch(w, "cuda")
plan = shuf.shuf_plan(w.n, w.elem_bytes, w.k, w.L, w.seed)
scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device="cuda")
for leaves in (1, 0, 1, 0):
    for _ in range(2):
        shuf.shuf_debug_run_levels(plan, x, scratch, 255, leaves)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        shuf.shuf_debug_run_levels(plan, x, scratch, 255, leaves)
    e1.record()
    torch.cuda.synchronize()
    print(f"run_leaves={leaves}: {e0.elapsed_time(e1) / 5:.3f} ms/run")
