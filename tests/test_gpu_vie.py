"""GPU parity of the VIE mode (src/vie.cpp) against the VIE oracle
(oracle/vie_oracle.py, pinned on the reference's tests/test_vie.cpp) and on the reference's own
test cases run through the device path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_03009_b200 import fus  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return fus.context(0)


@pytest.fixture(scope="module")
def vo():
    from oracle import vie_oracle
    return vie_oracle


def cube(lib, n, dx):
    return lib.make_grid([0, 0, 0], [n * dx] * 3, dx, 1)


def host(t):
    return t.cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_contrast_and_maps_vs_oracle(ctx, orc, vo):  # tests/test_vie.cpp:32-76
    g, go = cube(fus, 8, 1e-3), cube(orc, 8, 1e-3)
    w, lv = fus.medium_preset("water"), fus.medium_preset("liver")
    m = fus.slab_map(g, w, lv, 4e-3, 2e-3)
    mo = vo.slab_map(go, orc.medium_preset("water"), orc.medium_preset("liver"), 4e-3, 2e-3)
    assert np.array_equal(m.c, mo.c) and np.array_equal(m.beta, mo.beta)
    for n in (1, 2, 3):  # k^2 - kbar^2 cancels: compare to the operands' scale |kbar|^2, to ~1 ulp
        a, b = host(m.wavenumber_contrast(1.1e6, n)), mo.wavenumber_contrast(1.1e6, n)
        kb2 = abs(orc.complex_wavenumber(orc.medium_preset("water"), 1.1e6, n).k) ** 2
        assert np.array_equal(a == 0, b == 0)
        assert np.max(np.abs(a - b)) <= 4e-16 * kb2
    assert np.max(np.abs(host(fus.homogeneous_map(g, w).wavenumber_contrast(1.1e6, 2)))) == 0.0
    r = m.resample(g)
    assert np.array_equal(r.c, m.c) and np.array_equal(r.beta, m.beta)
    g2 = fus.make_grid([0.3e-3, 0.2e-3, 0.1e-3], [7.7e-3, 7.2e-3, 7.5e-3], 0.7e-3, 1)
    g2o = orc.VoxelGrid(g2.lo, g2.hi, g2.dx, g2.dims, 1)
    r, ro = m.resample(g2), mo.resample(g2o)
    assert np.array_equal(r.c, ro.c) and np.array_equal(r.beta, ro.beta)


def test_vie_operator_vs_oracle_16cubed(ctx, orc, vo):  # tests/test_vie.cpp:91-103
    g, go = cube(fus, 16, 0.2e-3), cube(orc, 16, 0.2e-3)
    k = fus.complex_wavenumber(fus.medium_preset("water"), 1.1e6, 1)
    ko = orc.Wavenumber(k.k, 1, k.omega)
    chi = fus.random_vector(g.count(), 42) * (0.05 * abs(k.k) ** 2)
    p = fus.random_vector(g.count(), 43)
    fast = host(fus.vie_operator_apply(p, chi, fus.GreenKernel(g, k)))
    dense = vo.dense_vie_matrix(ko, go, chi) @ p
    assert np.max(np.abs(fast - dense)) < 1e-12 * np.max(np.abs(dense))


def test_gmres_dense_system_and_failure(ctx):  # tests/test_vie.cpp:105-145
    rng = np.random.default_rng(7)
    n = 48
    A = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) * 0.1 + 3.0 * np.eye(n)
    Ad = torch.from_numpy(A).cuda()
    b = fus.random_vector(n, 9)
    sol = fus.gmres(lambda x: Ad @ x, b, 1e-12, 500, 20)
    x = host(sol.field)
    assert np.linalg.norm(A @ x - b) < 1e-11 * np.linalg.norm(b)
    assert sol.residual_history and sol.residual_history[-1] < 1e-12
    z = fus.gmres(lambda x: Ad @ x, np.zeros(n, np.complex128), 1e-12, 10)
    assert np.linalg.norm(host(z.field)) == 0.0
    S = np.zeros((64, 64), np.complex128)
    for i in range(64):
        S[i, (i + 1) % 64] = 1.0
    Sd = torch.from_numpy(S).cuda()
    e1 = np.zeros(64, np.complex128)
    e1[0] = 1.0
    with pytest.raises(fus.ConvergenceError) as e:
        fus.gmres(lambda x: Sd @ x, e1, 1e-14, 3, 3)
    assert e.value.residual_history
    with pytest.raises(ValueError):
        fus.gmres(lambda x: Ad @ x, b, 0.0, 10)


def test_solve_vie_zero_contrast_dense_and_oracle(ctx, orc, vo):  # tests/test_vie.cpp:147-172
    w = fus.medium_preset("water")
    k = fus.complex_wavenumber(w, 1.1e6, 1)
    g = cube(fus, 10, 0.3e-3)
    rhs = fus.random_vector(g.count(), 11)
    sol = fus.solve_vie(rhs, np.zeros(g.count(), np.complex128), fus.GreenKernel(g, k), 1e-10)
    assert np.max(np.abs(host(sol.field) - rhs)) < 1e-10 * np.max(np.abs(rhs)) and sol.iterations <= 1
    g, go = cube(fus, 9, 0.25e-3), cube(orc, 9, 0.25e-3)
    ko = orc.Wavenumber(k.k, 1, k.omega)
    chi = host(fus.slab_map(g, w, fus.medium_preset("liver"), 1.1e-3, 0.6e-3).wavenumber_contrast(1.1e6, 1))
    rhs = fus.random_vector(g.count(), 5)
    sol = fus.solve_vie(rhs, chi, fus.GreenKernel(g, k), 1e-10, 400)
    direct = np.linalg.solve(vo.dense_vie_matrix(ko, go, chi), rhs)
    assert np.linalg.norm(host(sol.field) - direct) < 1e-8 * np.linalg.norm(direct)
    ref = vo.solve_vie(rhs, chi, orc.GreenKernel(go, ko, workers=8), 1e-10, 400)
    assert sol.iterations == ref.iterations
    assert len(sol.residual_history) == len(ref.residual_history)
    assert np.allclose(sol.residual_history, ref.residual_history, rtol=1e-6, atol=1e-14)
    assert rel(host(sol.field), ref.field) < 1e-10


def test_weak_contrast_born(ctx):  # tests/test_vie.cpp:174-192
    g = cube(fus, 12, 0.2e-3)
    k = fus.complex_wavenumber(fus.medium_preset("water"), 1.1e6, 1)
    K = fus.GreenKernel(g, k)
    chi = np.zeros(g.count(), np.complex128)
    for iz in range(4, 8):
        for iy in range(4, 8):
            for ix in range(4, 8):
                chi[g.index(ix, iy, iz)] = 1e-3 * abs(k.k) ** 2
    rhs = fus.random_vector(g.count(), 21)
    x = host(fus.solve_vie(rhs, chi, K, 1e-12, 400).field)
    born = rhs + host(K.apply(chi * rhs))
    assert np.linalg.norm(x - born) / np.linalg.norm(rhs) < 1e-5
    assert np.linalg.norm(x - born) < 0.1 * np.linalg.norm(x - rhs)


def _tiny(lib, n_h):  # tests/test_vie.cpp:194-201
    t = lib.transducer_preset("H131", 15.0, 128)
    t.f0 = 0.25e6
    w = lib.medium_preset("water")
    return lib.CascadeConfig(w, t, lib.plan_nested_meshes(t, w, 6e-3, 3, n_h, 0.35), n_h)


def test_inhomogeneous_cascade_homogeneous_map_and_slab(ctx, orc, vo):  # tests/test_vie.cpp:194-233
    cfg = _tiny(fus, 3)
    homo = fus.run_cascade(cfg)
    m = fus.homogeneous_map(cfg.plan.for_harmonic(2).grid, fus.medium_preset("water"))
    inhomo = fus.run_cascade_inhomogeneous(cfg, m, fus.VieConfig(tol=1e-8))
    for n in (1, 2, 3):
        assert rel(host(inhomo.p(n).values), host(homo.p(n).values)) < 1e-6
    # a liver slab: against the oracle's inhomogeneous cascade (VIE solves at 1e-10)
    cfgo = _tiny(orc, 3)
    g2 = cfg.plan.for_harmonic(2).grid
    g2o = cfgo.plan.for_harmonic(2).grid
    ms = fus.slab_map(g2, fus.medium_preset("water"), fus.medium_preset("liver"), 20e-3, 4e-3)
    mso = vo.slab_map(g2o, orc.medium_preset("water"), orc.medium_preset("liver"), 20e-3, 4e-3)
    got = fus.run_cascade_inhomogeneous(cfg, ms, fus.VieConfig(tol=1e-10, max_iter=400))
    ref = vo.run_cascade_inhomogeneous(cfgo, mso, vo.VieConfig(tol=1e-10, max_iter=400), workers=8)
    assert got.source_normalization == pytest.approx(ref.source_normalization, rel=1e-12)
    for n in (1, 2, 3):
        assert got.p(n).grid.dims == ref.p(n).grid.dims
        assert rel(host(got.p(n).values), ref.p(n).values) < 1e-8, n
    base = host(homo.p(1).values)
    r1 = rel(host(got.p(1).values), base)
    assert 1e-3 < r1 < 0.5  # the slab scatters, as a perturbation
