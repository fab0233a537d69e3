"""Race probe: repeats GreenKernel builds and applies on one grid and counts distinct results
(bitwise). Usage: python tools/race_probe.py nx ny nz [builds] [applies_per_build]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402

nx, ny, nz = (int(a) for a in sys.argv[1:4])
builds = int(sys.argv[4]) if len(sys.argv) > 4 else 10
applies = int(sys.argv[5]) if len(sys.argv) > 5 else 20
dx = 1e-4
g = fus.make_grid([0, 0, 0], [nx * dx, ny * dx, nz * dx], dx, 4)
k = fus.complex_wavenumber(fus.medium_preset("water"), 0.8e6, 4)
f = torch.from_numpy(fus.random_vector(g.count(), 4)).cuda()
seen_build, seen_apply = {}, {}
ref = None
for b in range(builds):
    K = fus.GreenKernel(g, k)
    for a in range(applies):
        u = K.apply(f)
        h = hashlib.sha1(u.cpu().numpy().tobytes()).hexdigest()[:12]
        seen_apply[h] = seen_apply.get(h, 0) + 1
        if ref is None:
            ref = u.clone()
        elif a == 0:
            pass
    d = float((u - ref).abs().max() / ref.abs().max())
    seen_build[h] = seen_build.get(h, 0) + 1
    if d:
        print("build", b, "max rel diff", d)
    del K
print("padded", fus.padded_dims(g), "distinct applies", len(seen_apply), dict(sorted(seen_apply.items(), key=lambda x: -x[1])[:5]))
