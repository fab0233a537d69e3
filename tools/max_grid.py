"""Largest single-GPU apply: a 1024^3 grid (2048^3 circulant embedding, complex128; the
reference's own padded array alone would be 137 GB). Reports the device footprint, build and
apply times, and checks two sampled voxels against the oracle's direct sum
(direct_potential_oracle restricted to those voxels, src/potential.cpp:203-238)."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
c, f0 = 1540.0, 1.1e6
h = (c / f0) / 6.0
g = fus.make_grid([0, 0, 0], [n * h] * 3, h, 1)
k = fus.Wavenumber(complex(2 * math.pi * f0 / c, 0.0), 1, 2 * math.pi * f0)
t0 = time.perf_counter()
f = fus.random_vector(g.count(), 77)
gen_s = time.perf_counter() - t0
fd = torch.from_numpy(f).cuda()
free0, total = torch.cuda.mem_get_info()
t0 = time.perf_counter()
K = fus.GreenKernel(g, k)
torch.cuda.synchronize()
build_s = time.perf_counter() - t0
u = torch.empty_like(fd)
K.apply(fd, out=u)
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = 3
for _ in range(reps):
    K.apply(fd, out=u)
torch.cuda.synchronize()
apply_s = (time.perf_counter() - t0) / reps
free1, _ = torch.cuda.mem_get_info()
out = {"grid": list(g.dims), "padded": list(K.padded), "voxels": g.count(), "build_s": build_s,
       "apply_s": apply_s, "grid_pts_per_s": g.count() / apply_s,
       "device_gb_used_total": (total - free1) / 1e9, "kernel_device_gb": K.device_bytes() / 1e9 if hasattr(K, "device_bytes") else None,
       "host_rng_s": gen_s}
try:
    from oracle import fus_oracle as orc
    idx = np.array([0, g.count() // 2 + g.dims[0] // 3])
    got = u[torch.from_numpy(idx).cuda()].cpu().numpy()
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 1)
    t0 = time.perf_counter()
    ref = orc.direct_potential_at(orc.Wavenumber(k.k, 1, k.omega), go, f, idx)
    out["sampled_max_rel_err"] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    out["oracle_s"] = time.perf_counter() - t0
except ImportError:
    pass
print(json.dumps(out))
