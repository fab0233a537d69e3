"""Pins of the VIE oracle (oracle/vie_oracle.py, a restatement of src/vie.cpp): the reference's own
tests/test_vie.cpp cases, at the reference's sizes and tolerances, on CPU."""
import numpy as np
import pytest

from oracle import fus_oracle as orc
from oracle import vie_oracle as vie

WATER = orc.medium_preset("water")
LIVER = orc.medium_preset("liver")


def cube_grid(n, dx):  # tests/test_vie.cpp:23-26
    return orc.make_grid([0, 0, 0], [n * dx] * 3, dx, 1)


def test_medium_map_basics():  # tests/test_vie.cpp:32-76
    g = cube_grid(8, 1e-3)
    m = vie.homogeneous_map(g, WATER)
    assert m.is_homogeneous() and m.contrast_support().size == 0
    assert np.max(np.abs(m.wavenumber_contrast(1.1e6, 2))) == 0.0
    m = vie.slab_map(g, WATER, LIVER, 4e-3, 2e-3)
    assert not m.is_homogeneous()
    chi = m.wavenumber_contrast(1.1e6, 1)
    kb = orc.complex_wavenumber(WATER, 1.1e6, 1)
    xs = (np.arange(8) + 0.5) * 1e-3
    inside = np.broadcast_to((np.abs(xs - 4e-3) <= 1e-3)[None, None, :], (8, 8, 8)).reshape(-1)
    kx = complex(2 * np.pi * 1.1e6 / LIVER.c0, kb.k.imag)
    assert inside.sum() == 2 * 8 * 8 and m.contrast_support().size == 2 * 8 * 8
    assert np.all(m.c[inside] == LIVER.c0) and np.all(m.beta[inside] == LIVER.beta)
    assert np.all(np.abs(chi[inside] - (kx * kx - kb.k * kb.k)) < 1e-9 * abs(kb.k * kb.k))
    assert np.all(m.c[~inside] == WATER.c0) and np.all(chi[~inside] == 0)
    r = m.resample(g)
    assert np.max(np.abs(r.c - m.c)) < 1e-12 and np.max(np.abs(r.beta - m.beta)) < 1e-12


def test_vie_operator_matches_dense_assembly():  # tests/test_vie.cpp:91-103 (16^3)
    g = cube_grid(16, 0.2e-3)
    k = orc.complex_wavenumber(WATER, 1.1e6, 1)
    K = orc.GreenKernel(g, k, workers=8)
    chi = orc.random_vector(g.count(), 42) * (0.05 * abs(k.k) ** 2)
    p = orc.random_vector(g.count(), 43)
    fast = vie.vie_operator_apply(p, chi, K)
    slow = vie.dense_vie_matrix(k, g, chi) @ p
    assert np.max(np.abs(fast - slow)) < 1e-12 * np.max(np.abs(slow))


def _dense_system():  # tests/test_vie.cpp:105-116 (the same construction, numpy draws)
    rng = np.random.default_rng(7)
    n = 48
    A = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) * 0.1 + 3.0 * np.eye(n)
    return A, orc.random_vector(n, 9)


def test_gmres_dense_system_and_zero_rhs():
    A, b = _dense_system()
    sol = vie.gmres(lambda x: A @ x, b, 1e-12, 500, 20)
    assert np.linalg.norm(A @ sol.field - b) < 1e-11 * np.linalg.norm(b)
    assert sol.residual_history and sol.residual_history[-1] < 1e-12
    z = vie.gmres(lambda x: A @ x, np.zeros(48, np.complex128), 1e-12, 10)
    assert np.linalg.norm(z.field) == 0.0
    with pytest.raises(ValueError):
        vie.gmres(lambda x: A @ x, b, 0.0, 10)


def test_gmres_reports_non_convergence():  # tests/test_vie.cpp:129-145
    n = 64
    A = np.zeros((n, n), np.complex128)
    for i in range(n):
        A[i, (i + 1) % n] = 1.0
    b = np.zeros(n, np.complex128)
    b[0] = 1.0
    with pytest.raises(vie.ConvergenceError) as e:
        vie.gmres(lambda x: A @ x, b, 1e-14, 3, 3)
    assert e.value.residual_history


def test_solve_vie_zero_contrast_and_dense_direct():  # tests/test_vie.cpp:147-172
    g = cube_grid(10, 0.3e-3)
    k = orc.complex_wavenumber(WATER, 1.1e6, 1)
    K = orc.GreenKernel(g, k, workers=8)
    rhs = orc.random_vector(g.count(), 11)
    sol = vie.solve_vie(rhs, np.zeros(g.count(), np.complex128), K, 1e-10)
    assert np.max(np.abs(sol.field - rhs)) < 1e-10 * np.max(np.abs(rhs)) and sol.iterations <= 1
    g = cube_grid(9, 0.25e-3)
    K = orc.GreenKernel(g, k, workers=8)
    chi = vie.slab_map(g, WATER, LIVER, 1.1e-3, 0.6e-3).wavenumber_contrast(1.1e6, 1)
    rhs = orc.random_vector(g.count(), 5)
    sol = vie.solve_vie(rhs, chi, K, 1e-10, 400)
    direct = np.linalg.solve(vie.dense_vie_matrix(k, g, chi), rhs)
    assert np.linalg.norm(sol.field - direct) < 1e-8 * np.linalg.norm(direct)


def test_weak_contrast_born():  # tests/test_vie.cpp:174-192
    g = cube_grid(12, 0.2e-3)
    k = orc.complex_wavenumber(WATER, 1.1e6, 1)
    K = orc.GreenKernel(g, k, workers=8)
    chi = np.zeros(g.count(), np.complex128)
    for iz in range(4, 8):
        for iy in range(4, 8):
            for ix in range(4, 8):
                chi[g.index(ix, iy, iz)] = 1e-3 * abs(k.k) ** 2
    rhs = orc.random_vector(g.count(), 21)
    sol = vie.solve_vie(rhs, chi, K, 1e-12, 400)
    born = rhs + K.apply(chi * rhs)
    assert np.linalg.norm(sol.field - born) / np.linalg.norm(rhs) < 1e-5
    assert np.linalg.norm(sol.field - born) < 0.1 * np.linalg.norm(sol.field - rhs)


def _tiny_cfg(n_h):  # tests/test_vie.cpp:194-201
    t = orc.transducer_preset("H131", 15.0, 128)
    t.f0 = 0.25e6
    return orc.CascadeConfig(WATER, t, orc.plan_nested_meshes(t, WATER, 6e-3, 3, n_h, 0.35), n_h)


def test_homogeneous_map_reproduces_run_cascade():  # tests/test_vie.cpp:194-213
    cfg = _tiny_cfg(3)
    homo = orc.run_cascade(cfg, workers=8)
    m = vie.homogeneous_map(cfg.plan.for_harmonic(2).grid, WATER)
    inhomo = vie.run_cascade_inhomogeneous(cfg, m, vie.VieConfig(tol=1e-8), workers=8)
    for n in (1, 2, 3):
        a, b = inhomo.p(n).values, homo.p(n).values
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-6


def test_slab_scatters_as_a_perturbation():  # tests/test_vie.cpp:215-233
    cfg = _tiny_cfg(2)
    g2 = cfg.plan.for_harmonic(2).grid
    m = vie.slab_map(g2, WATER, LIVER, 20e-3, 4e-3)
    with_slab = vie.run_cascade_inhomogeneous(cfg, m, workers=8)
    base = orc.run_cascade(cfg, workers=8)
    rel = np.linalg.norm(with_slab.p(1).values - base.p(1).values) / np.linalg.norm(base.p(1).values)
    assert 1e-3 < rel < 0.5
