"""Runs the criterion-10 cascade (H101, water, 0.2 MHz, 5 harmonics, 256 sources) several times
in one process and reports, per harmonic, whether the fields are bitwise equal across runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03009_b200 import fus  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = fus.medium_preset("water")
t = fus.transducer_preset("H101", 100.0, 256)
t.f0 = 0.2e6
plan = fus.plan_nested_meshes(t, w, 10.2e-3, 6, 5)
for pg in plan.grids:
    print("grid", pg.harmonic, pg.grid.dims, fus.padded_dims(pg.grid))
runs = []
for r in range(reps):
    res = fus.run_cascade(fus.CascadeConfig(w, t, plan, 5))
    runs.append([res.p(n).values.cpu().numpy().copy() for n in range(1, 6)])
    print("run", r, "norm", res.source_normalization)
for n in range(5):
    diffs = [float(np.max(np.abs(runs[r][n] - runs[0][n])) / np.max(np.abs(runs[0][n]))) for r in range(reps)]
    print(f"p{n + 1}: max rel diff vs run 0 per run: {diffs}")
