"""GreenKernel build time (first build in the process, then a warm rebuild) at n^3 (cfg5: 768).
Usage: python tools/build_time_probe.py [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, math
from paper_2011_03009_b200 import fus
c, f0 = 1540.0, 1.1e6
h = (c / f0) / 6.0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
g = fus.make_grid([0, 0, 0], [n * h] * 3, h, 1)
k = fus.Wavenumber(complex(2 * math.pi * f0 / c, 0.0), 1, 2 * math.pi * f0)
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    K = fus.GreenKernel(g, k)
    torch.cuda.synchronize(); print(n, K.padded, 'build', time.perf_counter() - t0)
    del K
