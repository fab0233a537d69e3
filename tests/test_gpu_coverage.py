"""GPU parity coverage of the configurations and kernel lengths the benchmark runs.

* The static ladder: every padded length with compile-time-planned kernels, on every axis, is
  applied on a thin grid and checked against the oracle's apply (tools/ladder_check.py); the z
  axis runs twice, once under the default padding policy (warp-engine lengths preferred) and once
  with FUSG_PZ_WARP=0 so that every pass-C length is reached.
* The nested 5-harmonic solve exactly as bench.py times it (BASELINE config 4 geometry at the
  desk frequency, 4096 sources, padded x/y lengths 625/648/672 and z 768), stage by stage
  (src/cascade.cpp:42-107): p1 at sampled voxels against the oracle's monopole sum, then every
  p_n over its whole grid against the oracle's -apply(rhs_source(interpolated lower
  harmonics)) computed from the device's own lower harmonics, so errors cannot hide behind
  each other.  Tolerance: north_star's 1e-10 relative L2 per harmonic field.
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_03009_b200 import fus  # noqa: E402
from tools import cascades  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return fus.context(0)


def _ladder(axis, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ladder_check.py"), str(axis)],
                         capture_output=True, text=True, timeout=900, env=e)
    assert out.returncode == 0, out.stdout + out.stderr
    return {int(L): v for L, v in json.loads(out.stdout.strip().splitlines()[-1]).items()}


@pytest.mark.parametrize("axis,env", [(0, {"FUSG_PXY_FAST": "0"}), (1, {"FUSG_PXY_FAST": "0"}), (0, None),
                                      (2, None), (2, {"FUSG_PZ_WARP": "0"})])
def test_static_ladder_every_length_vs_oracle(ctx, axis, env):
    res = _ladder(axis, env)
    lens = fus.static_lengths(axis == 2)
    assert sorted(res) == sorted(lens)
    reached = {L: v for L, v in res.items() if v[0] is not None}
    if env:  # without the fast-length preference every ladder length is reachable
        assert sorted(reached) == sorted(lens), sorted(set(lens) - set(reached))
    else:  # default policies: at least the warp-engine and the largest lengths
        assert {512, 1536, 2048} <= set(reached)
    bad = {L: v for L, v in reached.items() if not v[1] <= 1e-12}
    assert not bad, bad


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_cfg4_desk_nested_solve_stage_by_stage(ctx, orc):
    cfg = cascades.cfg4(fus, desk=True)
    cfgo = cascades.cfg4(orc, desk=True)
    # the grids and padded boxes the bench's nested solve runs on
    grids = [cfg.plan.for_harmonic(i).grid for i in range(2, 6)]
    assert [tuple(g.dims) for g in grids] == [tuple(cfgo.plan.for_harmonic(i).grid.dims) for i in range(2, 6)]
    padded = [fus.padded_dims(g) for g in grids]
    assert {p[0] for p in padded} | {p[1] for p in padded} >= {625, 648, 672}
    assert {p[2] for p in padded} == {768}
    r = fus.run_cascade(cfg)
    med, medo, to = cfg.medium, cfgo.medium, cfgo.transducer
    k1o = orc.complex_wavenumber(medo, to.f0, 1)
    assert r.source_normalization == pytest.approx(orc.power_scale_factor(to, medo, k1o), rel=1e-12)
    # p1 on D2 at >= 200 sampled voxels (corners, face centres and random interior points)
    g2 = r.p(1).grid
    nx, ny, nz = g2.dims
    corners = [(x, y, z) for x in (0, nx - 1) for y in (0, ny - 1) for z in (0, nz - 1)]
    faces = [(0, ny // 2, nz // 2), (nx - 1, ny // 2, nz // 2), (nx // 2, 0, nz // 2), (nx // 2, ny - 1, nz // 2),
             (nx // 2, ny // 2, 0), (nx // 2, ny // 2, nz - 1), (nx // 2, ny // 2, nz // 2)]
    rng = np.random.default_rng(4)
    rnd = [tuple(int(v) for v in rng.integers(0, [nx, ny, nz])) for _ in range(200)]
    ijk = np.array(corners + faces + rnd)
    idx = ijk[:, 0] + nx * (ijk[:, 1] + ny * ijk[:, 2])
    pts = np.stack([g2.lo[a] + (ijk[:, a] + 0.5) * g2.dx for a in range(3)], 1)
    amp = r.source_normalization * to.cap_area() / float(len(to.source_points))
    got = r.p(1).values[torch.from_numpy(idx).cuda()].cpu().numpy()
    ref = orc.unnormalized_field(to, pts, k1o, amp)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-10
    # p2..p5 over their whole grids, each from the device's own lower harmonics
    host = [r.p(m).values.cpu().numpy() for m in range(1, 6)]
    ogrid = [orc.VoxelGrid(h.grid.lo, h.grid.hi, h.grid.dx, h.grid.dims, m + 1) for m, h in enumerate(r.harmonics)]
    errs = {}
    for i in range(2, 6):
        gi = ogrid[i - 1]
        lower = []
        for m in range(1, i):
            fld = orc.HarmonicField(ogrid[m - 1], host[m - 1], None)
            lower.append(fld if orc.same_grid(ogrid[m - 1], gi) else orc.interpolate(fld, gi))
        ki = orc.complex_wavenumber(medo, to.f0, i)
        rhs = orc.rhs_source(i, lower, medo, ki.omega)
        ref = -orc.GreenKernel(gi, ki, workers=os.cpu_count() or 1).apply(rhs)
        errs[i] = _rel_l2(host[i - 1], ref)
        del ref, rhs, lower
    assert all(e <= 1e-10 for e in errs.values()), errs
