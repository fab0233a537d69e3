"""Rayleigh/monopole sum on config 4's desk D2 grid (4096 sources) for ncu / terms-per-second."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_03009_b200 import fus
from tools import cascades

cfg = cascades.cfg4(fus, desk=True)
g = cfg.plan.for_harmonic(2).grid
fus.evaluate_first_harmonic(cfg.transducer, cfg.medium, g, 1.0)
torch.cuda.synchronize()
t0 = time.perf_counter()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    fus.evaluate_first_harmonic(cfg.transducer, cfg.medium, g, 1.0)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
terms = g.count() * len(cfg.transducer.source_points)
print(f"grid {g.dims} x {len(cfg.transducer.source_points)} sources: {dt*1e3:.1f} ms, {terms/dt:.3e} terms/s")
