"""Breaks the host-vector apply (fusg_kernel_apply_host) into PCIe copies and compute."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2011_03009_b200 import _lib, fus

g, k, f = bench.gpu_inputs(bench.CFG2)
K = fus.GreenKernel(g, k)
fh = torch.from_numpy(f).pin_memory()
uh = torch.empty_like(fh).pin_memory()
fd = torch.empty(f.size, dtype=torch.complex128, device="cuda")
for name, fn in [("h2d", lambda: fd.copy_(fh, non_blocking=True)), ("d2h", lambda: uh.copy_(fd, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt*1e3:.2f} ms  {fh.numel()*16/dt/1e9:.1f} GB/s")
L = _lib.lib()
for _ in range(2): _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
t0 = time.perf_counter()
for _ in range(10): _lib.check(L.fusg_kernel_apply_host(K.handle, fh.data_ptr(), uh.data_ptr(), 1.0))
print(f"apply_host: {(time.perf_counter()-t0)/10*1e3:.2f} ms")
