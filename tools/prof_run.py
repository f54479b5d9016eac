#!/usr/bin/env python
"""Run one (or --reps) shuffle(s) of a bench workload through the C ABI, for
ncu captures: `ncu ... python tools/prof_run.py hot`.  Exits non-zero on a
device error."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="hot")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
w = synth.WORKLOADS[a.workload]
dev = torch.device("cuda", 0)
d_off = None
if w.kind == "segmented":
    off = synth.segment_offsets(synth.c5_lengths(w.num_segments, w.seed))
    w = synth.Workload(w.name, int(off[-1]), w.elem_bytes, w.k, w.L, w.seed, w.kind, w.num_segments)
    x = synth.make_input_torch(w, dev, offsets=off)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
else:
    x = synth.make_input_torch(w, dev, n=a.n or None)
n = x.shape[0]
plan = shuf.shuf_plan(n, w.elem_bytes, w.k, w.L, w.seed)
scratch = torch.empty(plan.scratch_bytes if d_off is None else plan.scratch_bytes_segmented(d_off.numel() - 1),
                      dtype=torch.uint8, device=dev)
for _ in range(a.reps):
    if d_off is None:
        shuf.shuf_run(plan, x, scratch)
    else:
        shuf.shuf_segmented(plan, x, d_off, scratch)
err = shuf.shuf_last_device_error(plan)
print("launches", shuf.shuf_last_launch_count(plan), "device_error", err)
sys.exit(1 if err else 0)
