"""Kernel-spectrum build time (GreenKernel ctor, src/potential.cpp:72-118) for cubic grids.
Usage: python tools/build_times.py n1 [n2 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402

out = {}
for n in (int(a) for a in sys.argv[1:]):
    h = 1540.0 / 1.1e6 / 6
    g = fus.make_grid([0, 0, 0], [n * h] * 3, h, 1)
    k = fus.complex_wavenumber(fus.medium_preset("water"), 1.1e6, 1)
    fus.GreenKernel(g, k)  # warm-up (pool, module load)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        K = fus.GreenKernel(g, k)
        del K
    torch.cuda.synchronize()
    out[n] = {"padded": fus.padded_dims(g), "build_ms": round((time.perf_counter() - t0) / reps * 1e3, 3)}
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("FUSG_")}
print(json.dumps(out))
