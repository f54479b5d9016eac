"""Element-size sweep (the paper's Fig. 7, P:600-603,
P:665-671): one shuffle of n rows of eb bytes for eb in 1..64, our C-ABI path
(native kernels for 4/8/16 bytes, the gather route otherwise) against the
library GPU shuffles x[randperm(n)] and a sort by random 64-bit keys.
usage: python tools/sweep.py [log2 n] [reps]   -> one JSON line per size"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
from bench import gpu_baselines  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 1 << lg
dev = torch.device("cuda", 0)
k, L, seed = 256, 4096, 1
for eb in (1, 2, 4, 8, 16, 32, 64):
    x = torch.randint(0, 256, (n, eb), dtype=torch.uint8, device=dev)
    plan = shuf.shuf_plan(n, eb, k, L, seed)
    scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device=dev)
    for _ in range(2):
        shuf.shuf_run(plan, x, scratch)
    assert shuf.shuf_last_device_error(plan) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        shuf.shuf_run(plan, x, scratch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    line = {"eb": eb, "n": n, "route": "native" if eb in (4, 8, 16) else "gather", "ms": round(ms, 3),
            "elements_per_s": n / (ms / 1e3), "data_GBps": n * eb / (ms / 1e3) / 1e9,
            "baselines": gpu_baselines(x, n, ms, dev)}
    print(json.dumps(line), flush=True)
    del x, scratch, plan
    torch.cuda.empty_cache()
