"""Uninitialised-memory probe: fills most of the device memory with NaN through torch, returns
it to the driver, then runs the criterion-10 cascade through the library (whose stream-ordered
pool then reuses those pages) and compares every harmonic with a clean run saved by `save`.
Usage: python tools/poison_probe.py save|check [out.npz]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402

mode = sys.argv[1]
path = sys.argv[2] if len(sys.argv) > 2 else "/tmp/poison_ref.npz"
if mode == "check":
    free, _ = torch.cuda.mem_get_info()
    blocks = []
    for _ in range(64):
        n = int(free * 0.9) // 16 // 64
        t = torch.empty(n, dtype=torch.complex128, device="cuda")
        t.real.fill_(float("nan"))
        t.imag.fill_(float("nan"))
        blocks.append(t)
    torch.cuda.synchronize()
    del blocks, t
    torch.cuda.empty_cache()
w = fus.medium_preset("water")
t = fus.transducer_preset("H101", 100.0, 256)
t.f0 = 0.2e6
res = fus.run_cascade(fus.CascadeConfig(w, t, fus.plan_nested_meshes(t, w, 10.2e-3, 6, 5), 5))
fields = {f"p{n}": res.p(n).values.cpu().numpy() for n in range(1, 6)}
if mode == "save":
    np.savez(path, **fields)
    print("saved")
else:
    ref = np.load(path)
    for n in range(1, 6):
        a, b = fields[f"p{n}"], ref[f"p{n}"]
        print(f"p{n}: nan {int(np.isnan(a).sum())}, bitwise {np.array_equal(a, b)}, "
              f"max rel {float(np.nanmax(np.abs(a - b)) / np.max(np.abs(b))):.3e}")
