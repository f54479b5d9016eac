"""Per-kernel-class CUDA-event times of one warm shuffle (shuf_profile_run).
usage: python tools/ktime.py [workload] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
import synth  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "hot"
reps = 3
w = synth.WORKLOADS[wl]
dev = torch.device("cuda", 0)
d_off = None
if w.kind == "segmented":
    off = synth.segment_offsets(synth.c5_lengths(w.num_segments, w.seed))
    n = int(off[-1])
    x = synth.make_input_torch(w, dev, offsets=off)
    d_off = torch.as_tensor(off.astype("int64"), device=dev)
else:
    n = w.n
    x = synth.make_input_torch(w, dev)
plan = shuf.shuf_plan(n, w.elem_bytes, w.k, w.L, w.seed)
scratch = torch.empty(plan.scratch_bytes if d_off is None else plan.scratch_bytes_segmented(d_off.numel() - 1),
                      dtype=torch.uint8, device=dev)


INPLACE = "--inplace" in sys.argv
aux = torch.empty(max(1, shuf.shuf_aux_bytes_inplace(plan)), dtype=torch.uint8, device=dev) if INPLACE else None


def run():
    if INPLACE:
        shuf.shuf_run_inplace(plan, x, aux)
    elif d_off is None:
        shuf.shuf_run(plan, x, scratch)
    else:
        shuf.shuf_segmented(plan, x, d_off, scratch)


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
print(f"{wl}: {e0.elapsed_time(e1) / reps:.3f} ms/shuffle (stream-ordered, no per-launch events)"
      + (" IN-PLACE" if INPLACE else ""))
if INPLACE:
    print("aux MiB", shuf.shuf_aux_bytes_inplace(plan) / 2**20, "device error", shuf.shuf_last_device_error(plan))
    sys.exit(0)
prof = shuf.shuf_profile_run(plan, x, scratch, d_off)
for k, (ms, n) in prof.items():
    print(f"  {k:8s} {ms:8.3f} ms  launches={n}")
print("device error", shuf.shuf_last_device_error(plan), "env SHUF_FAST_FINISH =", os.environ.get("SHUF_FAST_FINISH"))
run()
c = shuf.shuf_debug_clocks(plan)
if "--scatter" in sys.argv:
    print("scatter CTA 0 level 0 tile phases (cycles): draws+count, wait+sync, scan, place, copyout, total")
    for it in range(1, 30):
        t = c[256 + it * 6: 256 + it * 6 + 6]
        if t[0] == 0:
            break
        nx = c[256 + (it + 1) * 6]
        print(f"  tile {it}: {t[1]-t[0]:6d} {t[2]-t[1]:6d} {t[3]-t[2]:6d} {t[4]-t[3]:6d} {t[5]-t[4]:6d}  total {nx - t[0] if nx else 0:6d}")
    sys.exit(0)
if int(os.environ.get("SHUF_DBG", "0")) & 4:
    print("pipelined finish CTA 0 per item (cycles): S count+scan, S place, S period; F FY, F period")
    for it in range(1, 30):
        t = c[it * 6: it * 6 + 5]
        if t[0] == 0:
            break
        n = c[(it + 1) * 6: (it + 1) * 6 + 5]
        print(f"  item {it}: S {t[1]-t[0]:6d} {t[2]-t[1]:6d} per {n[0]-t[0] if n[0] else 0:6d} | "
              f"F {t[4]-t[3]:6d} per {n[3]-t[3] if n[3] else 0:6d}")
    sys.exit(0)
if os.environ.get("SHUF_DBG") == "2":
    print("general finish CTA 0 per item (cycles): smem level, any_big+next load, FY(handle_children)+sync, store issue, total")
    for it in range(1, 30):
        t = c[it * 6: it * 6 + 5]
        if t[0] == 0:
            break
        nxt = c[(it + 1) * 6]
        print(f"  item {it}: {t[1]-t[0]:6d} {t[2]-t[1]:6d} {t[3]-t[2]:6d} {t[4]-t[3]:6d}  total {nxt - t[0] if nxt else 0:6d}")
    sys.exit(0)
print("fast-finish CTA 0 per item (cycles): scan+wait, place, partners, FY, FY||draws+count(next), store+rotate, total")
for it in range(1, 12):
    t = c[it * 6: it * 6 + 6]
    if t[0] == 0:
        break
    nxt = c[(it + 1) * 6]
    print(f"  item {it}: {t[1]-t[0]:6d} {t[2]-t[1]:6d} {t[3]-t[2]:6d} {t[4]-t[3]:6d} {t[5]-t[4]:6d} "
          f"{nxt - t[5] if nxt else 0:6d}  total {nxt - t[0] if nxt else 0:6d}")
