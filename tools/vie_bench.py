"""VIE solve throughput: solve_vie on the cfg2 grid (256^3, harmonic-2
wavenumber in attenuating water) with a liver slab across the box centre, tol 1e-6, restart 30.
Reports iterations and time per GMRES iteration; the CPU oracle (the reference's algorithm,
pocketfft apply) times a bounded sample of 2 iterations on the same problem."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402


def problem(lib, vie_mod, n=256):
    c, f0 = 1540.0, 1.1e6
    h = (c / (2 * f0)) / 6.0
    g = lib.make_grid([0, 0, 0], [n * h] * 3, h, 2)
    w = lib.medium_preset("water")
    k = lib.complex_wavenumber(w, f0, 2)
    m = vie_mod.slab_map(g, w, lib.medium_preset("liver"), 0.5 * n * h, 0.25 * n * h)
    return g, k, m


def run(cpu=True, n=256):
    g, k, m = problem(fus, fus, n)
    chi = m.wavenumber_contrast(1.1e6, 2)
    rhs = torch.from_numpy(fus.random_vector(g.count(), 17)).cuda()
    K = fus.GreenKernel(g, k)
    try:
        fus.solve_vie(rhs, chi, K, 1e-30, 2)  # warm-up (pool, modules)
    except fus.ConvergenceError:
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = fus.solve_vie(rhs, chi, K, 1e-6, 200, 30)
    dt = time.perf_counter() - t0
    out = {"grid": list(g.dims), "iterations": sol.iterations, "history_len": len(sol.residual_history),
           "final_residual": sol.residual_history[-1], "solve_s": dt,
           "ms_per_iteration": dt / max(1, len(sol.residual_history) - 1) * 1e3}
    if cpu:
        from oracle import fus_oracle as orc
        from oracle import vie_oracle as vo
        cores = os.cpu_count() or 1
        go, ko, mo = problem(orc, vo, n)
        Ko = orc.GreenKernel(go, ko, workers=cores)
        chio = mo.wavenumber_contrast(1.1e6, 2)
        rh = rhs.cpu().numpy()
        t0 = time.perf_counter()
        try:
            vo.solve_vie(rh, chio, Ko, 1e-30, 2, 30)
        except vo.ConvergenceError:
            pass
        ct = time.perf_counter() - t0
        out["cpu_baseline"] = {"ms_per_iteration": ct / 3 * 1e3, "cores": cores, "kind": "port",
                               "sample": "2 GMRES iterations (3 operator applies) by oracle/vie_oracle "
                                         "(pocketfft apply on the reference's 2N box)"}
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
