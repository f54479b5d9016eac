"""One in-place HOT shuffle (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2302_03317_b200 as shuf  # noqa: E402
import synth  # noqa: E402

w = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "hot"]
x = synth.make_input_torch(w, torch.device("cuda", 0))
shuf.inplace_shuffle(x, w.k, w.L, w.seed, elem_bytes=w.elem_bytes)
torch.cuda.synchronize()
print("ok")
