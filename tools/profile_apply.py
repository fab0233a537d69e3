"""Small driver for ncu: builds the cfg2 (256^3 -> 512^3) GreenKernel and runs a few applies.
Usage: python tools/profile_apply.py [n_side] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import fus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g, k, f = bench.gpu_inputs(bench.CFG2 if n == 256 else dict(bench.CFG5, n=n))
K = fus.GreenKernel(g, k)
fd = torch.from_numpy(f).cuda()
u = None
for _ in range(reps):
    u = K.apply(fd)
torch.cuda.synchronize()
print("ok", K.padded, float(u.abs().max()))
