"""Host-side cost of one device-resident apply call (C-ABI), against its GPU time.
Usage: python tools/step_host_time.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import _lib, fus  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ctx = fus.context(0)
g, k, f = bench.gpu_inputs(bench.CFG2)
K = fus.GreenKernel(g, k, ctx=ctx)
fd = torch.from_numpy(f).cuda()
ud = torch.empty_like(fd)
L = _lib.lib()
cs = torch.cuda.ExternalStream(ctx.stream_ptr)
for _ in range(5):
    _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))
ctx.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for n in (20, 50, steps):
    ctx.synchronize()
    ev0.record(cs)
    t0 = time.perf_counter()
    for _ in range(n):
        _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))
    host = (time.perf_counter() - t0) / n
    ev1.record(cs)
    ev1.synchronize()
    print(f"steps {n}: host {host * 1e3:.3f} ms/call, gpu {ev0.elapsed_time(ev1) / n:.3f} ms/step")
