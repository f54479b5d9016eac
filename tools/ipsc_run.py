"""One (or --reps) IpSc shuffle(s) of a workload through the C ABI (for ncu launch lists)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="hot")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
w = synth.WORKLOADS[a.workload]
if a.n:
    w = synth.Workload(w.name, a.n, w.elem_bytes, w.k, w.L, w.seed, w.kind, w.num_segments, w.note)
x = synth.make_input_torch(w, "cuda")
plan = shuf.shuf_plan(w.n, w.elem_bytes, w.k, w.L, w.seed)
aux = torch.empty(shuf.shuf_aux_bytes_ipsc(plan), dtype=torch.uint8, device="cuda")
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    shuf.shuf_run_ipsc(plan, x, aux)
    torch.cuda.synchronize()
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms, err {shuf.shuf_last_device_error(plan)}", flush=True)
if os.environ.get("SHUF_DBG"):
    c = shuf.shuf_debug_clocks(plan)[:8]
    names = ["load", "RS tree", "R+multinomial", "TwoSweep", "stash FY", "children", "store"]
    print("small-kernel phases (cycles):", {n: c[i + 1] - c[i] for i, n in enumerate(names)})
