"""evaluate_potential_at (src/potential.cpp:161-201) throughput at the reference's use: on-axis
nodes of a field on the cfg4-desk D2 grid (src/analysis.cpp:135,148,235), with the CPU oracle
(the reference's algorithm, OpenMP over points) on a bounded sample beside it."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402
from tools import cascades  # noqa: E402


def run(cpu_points=16):
    cfg = cascades.cfg4(fus, desk=True)
    g = cfg.plan.for_harmonic(2).grid
    k2 = fus.complex_wavenumber(cfg.medium, cfg.transducer.f0, 2)
    f = torch.from_numpy(fus.random_vector(g.count(), 4)).cuda()
    xs = g.lo[0] + (np.arange(g.dims[0]) + 0.5) * g.dx
    nodes = np.stack([xs, np.zeros_like(xs), np.zeros_like(xs)], 1)
    fus.evaluate_potential_at(k2, g, f, nodes[:8])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        v = fus.evaluate_potential_at(k2, g, f, nodes)
    dt = (time.perf_counter() - t0) / reps
    terms = g.count() * len(nodes)
    out = {"grid": list(g.dims), "points": len(nodes), "terms": terms, "ms": dt * 1e3,
           "terms_per_s": terms / dt}
    if cpu_points:
        from oracle import fus_oracle as orc
        cores = os.cpu_count() or 1
        orc.lib().orc_set_num_threads(cores)
        go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 2)
        fh = f.cpu().numpy()
        sel = nodes[:: max(1, len(nodes) // cpu_points)][:cpu_points]
        t0 = time.perf_counter()
        ref = orc.evaluate_potential_at(orc.Wavenumber(k2.k, 2, k2.omega), go, fh, sel)
        ct = time.perf_counter() - t0
        got = fus.evaluate_potential_at(k2, g, f, sel)
        out["cpu_baseline"] = {"terms_per_s": g.count() * len(sel) / ct, "cores": cores, "kind": "port",
                               "sample": f"{len(sel)} on-axis points x {g.count()} voxels (oracle, OpenMP over points)"}
        out["max_rel_diff_vs_oracle"] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
