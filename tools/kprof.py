"""Per-kernel-class split of one shuffle of n rows of eb bytes:
python tools/kprof.py n eb k L [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402

n, eb, k, L = (int(v) for v in sys.argv[1:5])
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 1
x = torch.randint(0, 256, (n, eb), dtype=torch.uint8, device="cuda")
plan = shuf.shuf_plan(n, eb, k, L, seed)
scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device="cuda")
shuf.shuf_run(plan, x, scratch)
for _ in range(2):
    prof = shuf.shuf_profile_run(plan, x, scratch)
print(f"n={n} eb={eb} k={k} L={L} S_fuse planned levels={plan.planned_levels}")
for c, (ms, cnt) in prof.items():
    print(f"  {c:8s} {ms:8.3f} ms  launches={cnt}")
print(shuf.shuf_last_run_stats(plan))
