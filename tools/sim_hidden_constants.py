#!/usr/bin/env python
"""Section 7 of the paper (Fig. 11) on the GPU: mean over RUNS
independent runs of R / sqrt(2 n k ln k) (Lemma 2) and M / (k sqrt(n k ln k))
(Corollary 5) from shuf_sim_rough_scatter (D9), plus M / (k sqrt n),
whose large-n limit for multinomial bucket sizes is the Brownian-bridge constant
sqrt(2/pi) * (1/k) sum_i sqrt(t_i (1 - t_i)) -> sqrt(2 pi)/8 = 0.3133.

    python tools/sim_hidden_constants.py [--runs 1000] [--out profiles/r02_hidden_constants.md]
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=1000)
ap.add_argument("--out", default="")
a = ap.parse_args()
rows = []
for k in (64, 256, 65536):
    for lg in (20, 22, 24, 26, 28):
        n = 1 << lg
        if k > 32768 and n // k > 30000:
            continue
        T = torch.zeros(a.runs, dtype=torch.int64, device="cuda")
        M = torch.zeros(a.runs, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        shuf.shuf_sim_rough_scatter(n, k, 2023, a.runs, T, M)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        R = n - T.cpu().numpy().astype(np.float64)
        Mv = M.cpu().numpy().astype(np.float64)
        lk = math.log(k)
        t = np.arange(1, k + 1) / k
        bridge = math.sqrt(2 / math.pi) * np.sqrt(t * (1 - t)).sum() / k
        rows.append((k, lg, R.mean() / math.sqrt(2 * n * k * lk), (R <= math.sqrt(2 * n * k * lk)).mean(),
                     Mv.mean() / (k * math.sqrt(n * k * lk)), Mv.mean() / (k * math.sqrt(n)), bridge, dt))
        print(rows[-1], flush=True)
lines = ["| k | n | mean R/sqrt(2nk ln k) | P[R <= bound] | mean M/(k sqrt(nk ln k)) | mean M/(k sqrt n) | bridge limit | GPU s |",
         "|---|---|---|---|---|---|---|---|"]
for k, lg, r, pr, m1, m2, br, dt in rows:
    lines.append(f"| {k} | 2^{lg} | {r:.4f} | {pr:.3f} | {m1:.5f} | {m2:.4f} | {br:.4f} | {dt:.3f} |")
txt = "\n".join(lines)
print(txt)
if a.out:
    with open(a.out, "w") as f:
        f.write(f"# Hidden-constant simulation (PAPER.md section 7, Fig. 11), {a.runs} runs per row, seed 2023\n\n")
        f.write("Produced by `python tools/sim_hidden_constants.py` on one B200 (shuf_sim_rough_scatter, DESIGN.md D9).\n\n")
        f.write(txt + "\n")
