"""Per-pass CUDA-event times of one GreenKernel apply on an arbitrary nx x ny x nz grid (cfg5's
wavenumber and spacing), e.g. the cascade grids. Usage: python tools/dims_times.py nx ny nz [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import _lib, fus  # noqa: E402

nx, ny, nz = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
h, kk, om = bench.geometry(bench.CFG5)
g = fus.make_grid([0, 0, 0], [nx * h, ny * h, nz * h], h, 1)
k = fus.Wavenumber(complex(kk, 0.0), 1, om)
f = torch.from_numpy(fus.random_vector(g.count(), 7)).cuda()
K = fus.GreenKernel(g, k)
u = torch.empty_like(f)
for _ in range(3):
    K.apply(f)
ms = (C.c_double * 5)()
_lib.check(_lib.lib().fusg_kernel_apply_timed(K.handle, f.data_ptr(), u.data_ptr(), 1.0, reps, ms))
per, tot = bench.algorithmic_bytes(g.dims, K.padded)
out = {"grid": list(g.dims), "padded": list(K.padded), "passes_ms": [round(m, 4) for m in ms],
       "total_ms": round(sum(ms), 4), "apply_GBps": round(tot / sum(ms) / 1e6, 1),
       "hbm_frac": round(tot / sum(ms) / 1e6 / bench.peaks()[0], 3),
       "env": {kk: v for kk, v in os.environ.items() if kk.startswith("FUSG_")}}
print(json.dumps(out))
