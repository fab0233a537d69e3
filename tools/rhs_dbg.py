import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math, numpy as np, torch
from paper_2011_03009_b200 import fus, _lib
import ctypes as C
w = fus.medium_preset("water")
g = fus.make_grid([0, 0, 0], [10e-3, 7e-3, 5e-3], 1e-3, 1)
omega = 2 * math.pi * 1.1e6
fields = [fus.random_vector(g.count(), 40 + i) for i in range(6)]
hf = [fus.HarmonicField(g, v, None) for v in fields]
print("argtypes", _lib.lib().fusg_rhs_source_full.argtypes)
for n in (2, 3, 4):
    a = fus.rhs_source_full(n, hf[: n - 1], w, omega).cpu().numpy()
    b = fus.rhs_source(n, hf[: n - 1], w, omega).cpu().numpy()
    print(n, "M=n-1 equal", np.array_equal(a, b))
    for M in range(n, 7):
        try:
            got = fus.rhs_source_full(n, hf[:M], w, omega).cpu().numpy()
            print(n, M, "ok")
        except Exception as e:
            print(n, M, "ERR", e); sys.exit(1)
