"""Timing comparison against the library FFT (north_star: "cuFFT is used only as a timing
comparison, never on the product path"): the reference's apply algorithm (src/potential.cpp:
120-151: zero-pad to the P box, 3D FFT, multiply by the P-box spectrum, inverse 3D FFT, 1/|P|,
crop) run on the GPU with torch.fft (cuFFT, complex128), against this framework's pruned
5-pass apply (fusg_kernel_apply) on the same grid and wavenumber.  The cuFFT spectrum is built
from the reference's own kernel fill (offset_of wrap, self term at offset 0), so the two
outputs are compared too.  Both are timed with CUDA events over back-to-back applies after
warm-up.
Usage: python tools/cufft_compare.py [out.json]   (cube sides 256 = cfg2, 384, 512)"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03009_b200 import fus  # noqa: E402


def kernel_fill(g, k, P, dev):
    """K on the P box (src/potential.cpp:84-114): offset_of wrap, vol G(dx |o|), self weight at 0."""
    def offs(n, p):
        m = torch.arange(p, device=dev, dtype=torch.float64)
        o = torch.where(m < n, m, torch.where(m > p - n, m - p, torch.full_like(m, float("nan"))))
        return o
    ox, oy, oz = offs(g.dims[0], P[0]), offs(g.dims[1], P[1]), offs(g.dims[2], P[2])
    r2 = oz[:, None, None] ** 2 + oy[None, :, None] ** 2 + ox[None, None, :] ** 2
    r = g.dx * torch.sqrt(r2)
    vol = g.dx ** 3
    K = (vol * torch.exp(-k.k.imag * r) / (4.0 * math.pi * r)) * torch.exp(1j * k.k.real * r)
    K = torch.nan_to_num(K.to(torch.complex128), nan=0.0)
    w0 = fus.self_weight(k, g.dx)
    K[0, 0, 0] = complex(w0)
    del r2, r
    return K


def time_events(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def run(n, reps=10):
    cfg = bench.CFG2 if n == 256 else dict(bench.CFG5, n=n)
    g, k, f = bench.gpu_inputs(cfg)
    dev = "cuda"
    N = g.dims
    K = fus.GreenKernel(g, k)
    fd = torch.from_numpy(f).to(dev)
    ud = torch.empty_like(fd)
    ours_ms = time_events(lambda: K.apply(fd, out=ud), reps)
    ours = ud.clone()
    del K
    torch.cuda.empty_cache()
    P = [2 * v for v in N]  # the reference's own box
    khat = torch.fft.fftn(kernel_fill(g, k, P, dev))
    f3 = fd.reshape(N[2], N[1], N[0])
    out = {}

    def lib_apply():
        work = torch.zeros((P[2], P[1], P[0]), dtype=torch.complex128, device=dev)
        work[: N[2], : N[1], : N[0]] = f3
        work = torch.fft.fftn(work)
        work *= khat
        work = torch.fft.ifftn(work, norm="forward")
        work /= float(P[0] * P[1] * P[2])
        out["u"] = work[: N[2], : N[1], : N[0]].contiguous().reshape(-1)

    lib_ms = time_events(lib_apply, reps)
    rel = float(torch.linalg.norm(out["u"] - ours) / torch.linalg.norm(out["u"]))
    cnt = g.count()
    res = {"grid": list(N), "reference_box": P, "ours_padded": list(fus.padded_dims(g)),
           "ours_ms": ours_ms, "cufft_ms": lib_ms, "speedup": lib_ms / ours_ms,
           "ours_grid_pts_per_s": cnt / (ours_ms * 1e-3), "cufft_grid_pts_per_s": cnt / (lib_ms * 1e-3),
           "rel_l2_ours_vs_cufft": rel}
    del khat, out, fd, ud, ours
    torch.cuda.empty_cache()
    return res


def main():
    sides = [256, 384, 512]
    res = {"device": torch.cuda.get_device_name(0),
           "what": "reference apply algorithm with torch.fft (cuFFT, c128) on the 2N box vs fusg_kernel_apply",
           "note": ("cfg5 (768^3, 1536^3 box) does not fit the library path: the spectrum and the "
                    "work array are 58 GB each and fftn needs an out-of-place buffer"),
           "configs": [run(n) for n in sides]}
    s = json.dumps(res, indent=1)
    print(s)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s + "\n")


if __name__ == "__main__":
    main()
