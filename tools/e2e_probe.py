"""Host-vector apply (fusg_kernel_apply_host) on pageable and pinned buffers against the raw
PCIe copies and a host memcpy, for one bench workload.
Usage: python tools/e2e_probe.py [n_side (256 = cfg2, 768 = cfg5)] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import _lib, fus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g, k, f = bench.gpu_inputs(bench.CFG2 if n == 256 else dict(bench.CFG5, n=n))
K = fus.GreenKernel(g, k)
out = {"n": n, "bytes_each_way": f.nbytes, "env": {kk: v for kk, v in os.environ.items() if kk.startswith("FUSG_")}}
fh = torch.from_numpy(f).pin_memory()
uh = torch.empty_like(fh).pin_memory()
fd = torch.empty(f.size, dtype=torch.complex128, device="cuda")


def timed(fn, r=reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(r):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / r


out["h2d_pinned_GBps"] = f.nbytes / timed(lambda: fd.copy_(fh, non_blocking=True)) / 1e9
out["d2h_pinned_GBps"] = f.nbytes / timed(lambda: uh.copy_(fd, non_blocking=True)) / 1e9
dst = np.empty_like(f)
out["host_memcpy_1thread_GBps"] = f.nbytes / timed(lambda: np.copyto(dst, f), 2) / 1e9
L = _lib.lib()
out["apply_host_pinned_ms"] = 1e3 * timed(lambda: _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0)))
u = np.empty_like(f)
out["apply_host_pageable_ms"] = 1e3 * timed(lambda: K.apply_host(f, out=u))
out["bitwise_equal"] = bool(np.array_equal(u, uh.numpy()))
print(json.dumps(out))
