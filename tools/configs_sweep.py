"""Every BASELINE.json configuration on one B200, through the public API (fus mirror over the
C-ABI): apply throughput for cfg1 / cfg2 / cfg5, full cascades for cfg3 and cfg4 (desk
frequency; the 1.1 MHz cfg4 needs a ~2e9-voxel D2 grid whose 2N embedding does not fit one GPU,
DESIGN.md section 7).  Synthetic seeded inputs (mt19937 + U[-1, 1]).
Usage: python tools/configs_sweep.py [out.json]"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import fus  # noqa: E402
from tools import cascades  # noqa: E402


def apply_rate(g, k, f, steps):
    t0 = time.perf_counter()
    K = fus.GreenKernel(g, k)
    build_first = time.perf_counter() - t0
    t0 = time.perf_counter()
    K2 = fus.GreenKernel(g, k)
    torch.cuda.synchronize()
    build_warm = time.perf_counter() - t0
    del K2
    fd = torch.from_numpy(f).cuda()
    for _ in range(3):
        u = K.apply(fd)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cs = torch.cuda.ExternalStream(fus.context().stream_ptr)
    ev0.record(cs)
    for _ in range(steps):
        u = K.apply(fd)
    ev1.record(cs)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    n = g.count()
    out = {"grid": list(g.dims), "padded": list(K.padded), "ms_per_apply": ms, "grid_pts_per_s": n / (ms * 1e-3),
           "kernel_build_first_s": build_first, "kernel_build_warm_s": build_warm,
           "u_max_abs": float(u.abs().max())}
    del K, fd, u
    torch.cuda.empty_cache()
    return out


def cascade(cfg):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fus.run_cascade(cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"solve_s": wall, "grids": [list(h.grid.dims) for h in r.harmonics],
            "voxels": [h.grid.count() for h in r.harmonics],
            "peak_pa": [float(h.values.abs().max()) for h in r.harmonics],
            "rows": [t.__dict__ for t in r.timings]}


def main():
    res = {"device": torch.cuda.get_device_name(0), "data": "synthetic, seeded"}
    c = 1540.0
    # cfg1: 64^3, h = lambda/6 at 1.1 MHz, k = 2 pi f / c, iid U[-1, 1] seed 1234
    f0 = 1.1e6
    h = (c / f0) / 6.0
    g = fus.make_grid([0, 0, 0], [64 * h] * 3, h, 1)
    k = fus.Wavenumber(complex(2 * math.pi * f0 / c, 0.0), 1, 2 * math.pi * f0)
    res["cfg1"] = apply_rate(g, k, fus.random_vector(g.count(), 1234), 200)
    # cfg2: the bench workload
    g, k, f = bench.gpu_inputs(bench.CFG2)
    res["cfg2"] = apply_rate(g, k, f, 100)
    # cfg5: 768^3 at 6 points per wavelength (harmonic-1 wavenumber), iid U[-1, 1]
    h = (c / f0) / 6.0
    g = fus.make_grid([0, 0, 0], [768 * h] * 3, h, 1)
    k = fus.Wavenumber(complex(2 * math.pi * f0 / c, 0.0), 1, 2 * math.pi * f0)
    res["cfg5"] = apply_rate(g, k, fus.random_vector(g.count(), 5), 5)
    torch.cuda.empty_cache()
    # cfg3: uniform-grid 3-harmonic recursion (single mesh, h = lambda3 / 6)
    res["cfg3"] = cascade(cascades.cfg3(fus, 4096))
    torch.cuda.empty_cache()
    # cfg4 at the desk frequency (0.275 MHz, same geometry ratios)
    res["cfg4_desk"] = cascade(cascades.cfg4(fus, desk=True, n_points=4096))
    line = json.dumps(res)
    print(line)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
