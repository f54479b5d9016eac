import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle
import paper_2302_03317_b200 as shuf
for n, k, seed, runs in [(100003, 64, 3, 6), (5000, 64, 3, 4), (8192, 64, 3, 4), (4097, 64, 3, 4), (1 << 20, 256, 4, 4)]:
    T = torch.zeros(runs, dtype=torch.int64, device="cuda"); M = torch.zeros(runs, dtype=torch.int64, device="cuda")
    shuf.shuf_sim_rough_scatter(n, k, seed, runs, T, M); torch.cuda.synchronize()
    eT, eM = oracle.sim_rough_scatter(n, k, seed, runs)
    print(n, k, "gpu T", T.cpu().numpy().tolist(), "ora T", eT.tolist())
    print(n, k, "gpu M", M.cpu().numpy().tolist(), "ora M", eM.tolist())
