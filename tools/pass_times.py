"""Per-pass CUDA-event timings of one GreenKernel apply on an n^3 cube (bench workloads: 768 =
cfg5, 256 = cfg2; other sides use cfg5's wavenumber and h).
Usage: python tools/pass_times.py [n_side] [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import _lib, fus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.CFG2 if n == 256 else dict(bench.CFG5, n=n)
g, k, f = bench.gpu_inputs(cfg)
K = fus.GreenKernel(g, k)
fd = torch.from_numpy(f).cuda()
ud = torch.empty_like(fd)
for _ in range(3):
    K.apply(fd)
ms = (C.c_double * 5)()
_lib.check(_lib.lib().fusg_kernel_apply_timed(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, reps, ms))
per, tot = bench.algorithmic_bytes(g.dims, K.padded)
out = {name: {"ms": round(m, 4), "GBps": round(b / m / 1e6, 1)} for (name, b), m in zip(per.items(), ms)}
out["total_ms"] = round(sum(ms), 4)
out["u_checksum"] = [float(ud.real.sum()), float(ud.imag.sum()), float(ud.abs().max())]
out["apply_GBps"] = round(tot / sum(ms) / 1e6, 1)
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("FUSG_")}
print(json.dumps(out))
