"""Run the BASELINE bowl cascades (cfg3, cfg4 desk) on the GPU and print stage timings.
Usage: python tools/run_cascade.py [cfg3|cfg4desk|cfg4] [n_points]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_03009_b200 import fus
from tools import cascades

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4desk"
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = cascades.cfg3(fus, npts) if name == "cfg3" else cascades.cfg4(fus, desk=(name != "cfg4"), n_points=npts)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = fus.run_cascade(cfg)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
out = {"config": name, "n_points": npts, "wall_s": wall, "source_normalization": r.source_normalization,
       "grids": [list(h.grid.dims) for h in r.harmonics],
       "peak_pa": [float(h.values.abs().max()) for h in r.harmonics],
       "rows": [t.__dict__ for t in r.timings]}
print(json.dumps(out))
