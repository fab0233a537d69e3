"""Parity of every padded length with compile-time-planned kernels ("the static ladder"): for each
length L of fus.static_lengths() on one axis, a thin grid whose padded extent on that axis is L
(n valid points, the other two axes 3 and 2) is applied on the GPU and checked against the CPU
oracle's GreenKernel::apply (src/potential.cpp:120-151) on the reference's own 2N box.
Prints one JSON object {L: [n, rel_l2]} (n = null when no grid size pads to L on this axis
under the current padding policy, e.g. FUSG_PZ_WARP).
Usage: python tools/ladder_check.py axis   (0 = x, 1 = y, 2 = z)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import fus_oracle as orc  # noqa: E402
from paper_2011_03009_b200 import fus  # noqa: E402


def grid_for(L, axis, dx):
    """The largest n whose padded extent on `axis` is L (None if none within reach)."""
    for n in range((L + 1) // 2, max(0, (L + 1) // 2 - 64), -1):
        dims = [3, 2, 2] if axis != 1 else [2, 3, 2]
        dims[axis] = n
        g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
        if tuple(g.dims) == tuple(dims) and fus.padded_dims(g)[axis] == L:
            return g, dims
    return None, None


def main():
    axis = int(sys.argv[1])
    dx = 1e-4
    k = fus.complex_wavenumber(fus.medium_preset("water"), 1.1e6, 2)
    ko = orc.complex_wavenumber(orc.medium_preset("water"), 1.1e6, 2)
    out = {}
    for L in fus.static_lengths(axis == 2):
        g, dims = grid_for(L, axis, dx)
        if g is None:
            out[L] = [None, None]
            continue
        f = fus.random_vector(g.count(), 1000 + L)
        u = fus.GreenKernel(g, k).apply(f).cpu().numpy()
        go = orc.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
        ref = orc.GreenKernel(go, ko).apply(f)
        out[L] = [dims[axis], float(np.linalg.norm(u - ref) / np.linalg.norm(ref))]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
