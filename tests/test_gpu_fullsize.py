"""GPU parity at BASELINE.json's full sizes, where the CPU oracle cannot run the whole problem.

* cfg5: one 768^3 apply (1536^3 embedding, the L = 1536 kernels) against the oracle's direct sum
  (direct_potential_oracle, src/potential.cpp:203-238) at >= 64 sampled voxels (corners, face
  centres, random interior), plus the exact
  scaling property apply(2 f) == 2 apply(f) bit for bit.
* cfg3: the full uniform-grid 3-harmonic recursion (1.2e8 voxels, 4096 sources). Each stage is
  checked given the device's previous stage, so errors cannot hide behind each other:
  * p1 against the oracle's monopole sum at sampled voxels;
  * p2 and p3 against the oracle's direct volume sum of the oracle rhs_source
    (src/cascade.cpp:21-40) built from the downloaded lower harmonics.

Tolerance: north_star's 1e-10, taken per sampled voxel relative to the largest sampled
magnitude.
"""
import math
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_03009_b200 import fus  # noqa: E402
from tools import cascades  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return fus.context(0)


def _sample(dims, n, seed):
    """Flat indices of the 8 corners, the 6 face centres, the centre and n random voxels."""
    nx, ny, nz = dims
    pts = [(x, y, z) for x in (0, nx - 1) for y in (0, ny - 1) for z in (0, nz - 1)]
    pts += [(0, ny // 2, nz // 2), (nx - 1, ny // 2, nz // 2), (nx // 2, 0, nz // 2), (nx // 2, ny - 1, nz // 2),
            (nx // 2, ny // 2, 0), (nx // 2, ny // 2, nz - 1), (nx // 2, ny // 2, nz // 2)]
    rng = np.random.default_rng(seed)
    ijk = np.concatenate([np.array(pts), rng.integers(0, [nx, ny, nz], size=(n, 3))])
    return np.unique(ijk[:, 0] + nx * (ijk[:, 1] + ny * ijk[:, 2]))


def _close(got, ref, tol=1e-10):
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err <= tol, err
    return err


def test_cfg5_768cubed_apply_at_sampled_voxels(ctx, orc):
    # BASELINE config 5: 768^3 grid, k at 6 points per wavelength, iid U[-1,1] complex source
    c, f0 = 1540.0, 1.1e6
    h = (c / f0) / 6.0
    g = fus.make_grid([0, 0, 0], [768 * h] * 3, h, 1)
    assert g.dims == (768, 768, 768)
    k = fus.Wavenumber(complex(2 * math.pi * f0 / c, 0.0), 1, 2 * math.pi * f0)
    f = fus.random_vector(g.count(), 5150)
    K = fus.GreenKernel(g, k)
    assert K.padded == (1536, 1536, 1536)
    fd = torch.from_numpy(f).cuda()
    u = K.apply(fd)
    # exact: scaling the source by 2 scales every rounding step by 2
    assert torch.equal(K.apply(fd * 2.0), u * 2.0)
    idx = _sample(g.dims, 56, 7)
    assert idx.size >= 64
    got = u[torch.from_numpy(idx).cuda()].cpu().numpy()
    del u, fd
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 1)
    ref = orc.direct_potential_at(orc.Wavenumber(k.k, 1, k.omega), go, f, idx)
    _close(got, ref)


def test_cfg3_full_cascade_stage_by_stage(ctx, orc):
    cfg = cascades.cfg3(fus)
    cfgo = cascades.cfg3(orc)
    r = fus.run_cascade(cfg)
    g = r.p(2).grid
    assert g.count() > 1.0e8
    med, medo, t, to = cfg.medium, cfgo.medium, cfg.transducer, cfgo.transducer
    k1o = orc.complex_wavenumber(medo, to.f0, 1)
    assert k1o.k.imag > 0.0  # attenuating water: the complex-k paths
    assert r.source_normalization == pytest.approx(orc.power_scale_factor(to, medo, k1o), rel=1e-12)
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 2)
    idx = _sample(g.dims, 56, 11)
    assert idx.size >= 64
    ix, iy, iz = idx % g.dims[0], (idx // g.dims[0]) % g.dims[1], idx // (g.dims[0] * g.dims[1])
    pts = np.stack([g.lo[0] + (ix + 0.5) * g.dx, g.lo[1] + (iy + 0.5) * g.dx, g.lo[2] + (iz + 0.5) * g.dx], 1)
    sel = torch.from_numpy(idx).cuda()
    # p1: Rayleigh sum at the sampled voxel centres
    amp = r.source_normalization * to.cap_area() / float(len(to.source_points))
    _close(r.p(1).values[sel].cpu().numpy(), orc.unnormalized_field(to, pts, k1o, amp))
    # p2, p3: -apply_{k_n}(rhs_n) with rhs_n from the device's lower harmonics
    omega = 2 * math.pi * to.f0
    lower = [orc.HarmonicField(go, r.p(1).values.cpu().numpy(), None)]
    for n in (2, 3):
        rhs = orc.rhs_source(n, lower, medo, omega)
        kn = orc.complex_wavenumber(medo, to.f0, n)
        ref = -orc.direct_potential_at(kn, go, rhs, idx)
        pn = r.p(n).values
        _close(pn[sel].cpu().numpy(), ref)
        lower.append(orc.HarmonicField(go, pn.cpu().numpy(), None))
