import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2011_03009_b200 import _lib, fus
g, k, f = bench.gpu_inputs(bench.CFG2)
K = fus.GreenKernel(g, k)
fd = torch.from_numpy(f).cuda(); ud = torch.empty_like(fd)
L = _lib.lib(); ctx = K.ctx
def step(): _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), ud.data_ptr(), 1.0, None))
for _ in range(5): step()
ctx.synchronize()
cs = torch.cuda.ExternalStream(ctx.stream_ptr)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time
for n in (20, 100):
    ctx.synchronize(); e0.record(cs); t0=time.perf_counter()
    for _ in range(n): step()
    t1=time.perf_counter(); e1.record(cs); e1.synchronize()
    print(json.dumps({"env": os.environ.get("FUSG_COLROW_PP"), "n": n, "ms_per_step": e0.elapsed_time(e1)/n, "host_ms_per_call": (t1-t0)/n*1e3}))
