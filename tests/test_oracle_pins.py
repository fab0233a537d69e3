"""Pin the CPU oracle against the reference's own known-answer tests and recorded goldens.

Every case restates a reference test (file:line under /root/reference/proj) with the same
inputs and tolerance.  The oracle is trusted for GPU parity only because these pass.
"""
import math

import numpy as np
import pytest


def water(orc):
    return orc.medium_preset("water")


# ------------------------------------------------------------------ potential (test_potential.cpp)
def test_green_function_basics(orc):  # tests/test_potential.cpp:26-38
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    x, y = np.zeros(3), np.array([1e-3, 2e-3, -2e-3])
    r = np.linalg.norm(x - y)
    g = orc.green_function(x, y, k)
    assert abs(abs(g) - math.exp(-k.k.imag * r) / (4 * math.pi * r)) <= 1e-13 * abs(g)
    assert orc.green_function(y, x, k) == g
    with pytest.raises(ValueError):
        orc.green_function(x, x, k)


def test_equivalent_sphere_radius(orc):  # tests/test_potential.cpp:40-46
    assert orc.equivalent_sphere_radius(1.0) == pytest.approx(0.6203504908994001, rel=1e-12)
    dx = 45e-6
    a = orc.equivalent_sphere_radius(dx)
    assert 4.0 / 3.0 * math.pi * a ** 3 == pytest.approx(dx ** 3, rel=1e-12)


def _self_weight_simpson(k, a, n=4000):  # tests/oracles.hpp:37-45
    f = lambda r: np.exp(1j * k * r) * r
    h = a / n
    j = np.arange(1, n)
    s = f(0.0) + f(a) + np.sum(np.where(j % 2 == 1, 4.0, 2.0) * f(j * h))
    return s * h / 3.0


def test_self_weight_matches_sphere_integral(orc):  # tests/test_potential.cpp:48-59
    dx = 1e-4
    a = orc.equivalent_sphere_radius(dx)
    for n in (1, 3, 5):
        k = orc.complex_wavenumber(water(orc), 1.1e6, n)
        w = orc.self_weight(k, dx)
        ref = _self_weight_simpson(k.k, a)
        assert abs(w - ref) < 1e-10 * abs(ref)


def test_self_weight_series_branches(orc):  # tests/test_potential.cpp:61-73
    k = orc.Wavenumber(complex(10.0, 0.5), 1, 2 * math.pi * 1.1e6)
    dx = 1e-7
    a = orc.equivalent_sphere_radius(dx)
    assert abs(orc.self_weight(k, dx) - _self_weight_simpson(k.k, a)) < 1e-12 * a * a
    k0 = orc.Wavenumber(0j, 1, 1.0)
    w0 = orc.self_weight(k0, 1.0)
    assert w0.real == pytest.approx(0.5 * orc.equivalent_sphere_radius(1.0) ** 2, rel=1e-12)
    assert w0.imag == pytest.approx(0.0)


@pytest.mark.parametrize("seed,pad", [(1234, False), (1234, True), (2024, False)])
def test_fft_apply_matches_direct_20x18x16(orc, seed, pad):
    # tests/test_potential.cpp:75-92 (seed 1234, + small-prime subcase);
    # tests/acceptance.cpp:98-112 criterion 2 (seed 2024)
    g = orc.make_grid([0, 0, 0], [20e-4, 18e-4, 16e-4], 1e-4, 2)
    assert g.dims == (20, 18, 16)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 2)
    f = orc.random_vector(g.count(), seed)
    u = orc.GreenKernel(g, k, pad).apply(f)
    ref = orc.direct_potential_oracle(k, g, f)
    assert np.max(np.abs(u - ref)) < 1e-12 * np.max(np.abs(ref))


def test_any_padding_at_least_2n_minus_1_is_exact(orc):
    # src/potential.cpp:88-94: offset_of needs only P >= 2N-1 for the offsets (-N, N) to be
    # distinct; the GPU path pads to smooth sizes on that basis.
    g = orc.make_grid([0, 0, 0], [20e-4, 18e-4, 16e-4], 1e-4, 2)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 2)
    f = orc.random_vector(g.count(), 1234)
    ref = orc.direct_potential_oracle(k, g, f)
    for P in [(39, 35, 31), (42, 36, 35), (48, 45, 40)]:
        u = orc.GreenKernel(g, k, padded=P).apply(f)
        assert np.max(np.abs(u - ref)) < 1e-12 * np.max(np.abs(ref))


def test_apply_linear_and_translation_covariant(orc):  # tests/test_potential.cpp:94-115
    g = orc.make_grid([-3e-3, 1e-3, 0], [2e-3, 6e-3, 4e-3], 5e-4, 1)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    K = orc.GreenKernel(g, k)
    f, h = orc.random_vector(g.count(), 7), orc.random_vector(g.count(), 8)
    a = complex(0.3, -1.7)
    lhs = K.apply(a * f + h)
    rhs = a * K.apply(f) + K.apply(h)
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(rhs))
    off = np.array([11e-3, -4e-3, 9e-3])
    g2 = orc.VoxelGrid(g.lo + off, g.hi + off, g.dx, g.dims, g.harmonic)
    K2 = orc.GreenKernel(g2, k)
    u = K.apply(f)
    assert np.max(np.abs(K2.apply(f) - u)) < 1e-12 * np.max(np.abs(u))


def test_delta_reproduces_kernel_column(orc):  # tests/test_potential.cpp:117-139
    g = orc.make_grid([0, 0, 0], [9e-4, 8e-4, 7e-4], 1e-4, 1)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    K = orc.GreenKernel(g, k)
    delta = np.zeros(g.count(), np.complex128)
    j = g.index(4, 3, 2)
    delta[j] = 1.0
    col = K.apply(delta)
    vol = g.dx ** 3
    xj = g.center(4, 3, 2)
    for iz in range(g.dims[2]):
        for iy in range(g.dims[1]):
            for ix in range(g.dims[0]):
                i = g.index(ix, iy, iz)
                want = (orc.self_weight(k, g.dx) if i == j
                        else vol * orc.green_function(g.center(ix, iy, iz), xj, k))
                assert abs(col[i] - want) < 1e-13 * abs(want) + 1e-20


def test_helmholtz_residual_second_order(orc):  # tests/test_potential.cpp:141-181
    k = orc.complex_wavenumber(water(orc), 0.5e6, 1)
    probe = np.array([2.5e-3] * 3)
    source = np.array([0.5e-3] * 3)

    def residual(dx, n):
        g = orc.make_grid([0, 0, 0], [n * dx] * 3, dx, 1, probe)
        f = np.zeros(g.count(), np.complex128)
        s = [int(round((source[a] - g.lo[a]) / dx - 0.5)) for a in range(3)]
        f[g.index(*s)] = 1.0 / dx ** 3
        u = orc.GreenKernel(g, k).apply(f)
        c = [int(round((probe[a] - g.lo[a]) / dx - 0.5)) for a in range(3)]
        U = lambda i, j, l: u[g.index(i, j, l)]
        lap = (U(c[0] + 1, c[1], c[2]) + U(c[0] - 1, c[1], c[2]) + U(c[0], c[1] + 1, c[2]) +
               U(c[0], c[1] - 1, c[2]) + U(c[0], c[1], c[2] + 1) + U(c[0], c[1], c[2] - 1) -
               6.0 * U(*c)) / dx ** 2
        return abs(lap + k.k * k.k * U(*c))

    ratio = residual(2.0e-4, 16) / residual(1.0e-4, 32)
    assert 3.0 < ratio < 5.5


def test_off_grid_evaluation_matches_apply(orc):  # tests/test_potential.cpp:183-208
    g = orc.make_grid([0, 0, 0], [7e-4, 6e-4, 5e-4], 1e-4, 1)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 2)
    f = orc.random_vector(g.count(), 99)
    u = orc.GreenKernel(g, k).apply(f)
    pts, idx = [], []
    for iz in range(0, g.dims[2], 2):
        for iy in range(0, g.dims[1], 3):
            for ix in range(0, g.dims[0], 2):
                pts.append(g.center(ix, iy, iz))
                idx.append(g.index(ix, iy, iz))
    v = orc.evaluate_potential_at(k, g, f, pts)
    assert np.max(np.abs(v - u[idx])) < 1e-12 * np.max(np.abs(u))


def test_direct_oracle_refuses_oversized(orc):  # tests/test_potential.cpp:210-215
    g = orc.make_grid([0, 0, 0], [1.0, 1.0, 1.0], 1.0 / 64, 1)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    with pytest.raises(ValueError):
        orc.direct_potential_oracle(k, g, np.zeros(g.count(), np.complex128))


# ------------------------------------------------------------------ medium (test_medium.cpp)
def test_medium_presets_and_wavenumber(orc):  # tests/test_medium.cpp:11-60
    w = water(orc)
    assert (w.rho0, w.c0, w.beta, w.alpha0, w.eta) == (1000.0, 1480.0, 3.5, 0.2, 2.0)
    assert orc.attenuation_np_per_m(w, 1.1e6) == pytest.approx(0.2 * 1.1 * 1.1 / orc.K_DB_PER_NEPER,
                                                               rel=1e-14)
    liver = orc.medium_preset("liver")
    k1 = orc.complex_wavenumber(liver, 1.1e6, 1)
    k4 = orc.complex_wavenumber(liver, 1.1e6, 4)
    assert k1.k.real == pytest.approx(2 * math.pi * 1.1e6 / liver.c0, rel=1e-14)
    assert k4.k.real == pytest.approx(4 * k1.k.real, rel=1e-14)
    assert k4.k.imag / k1.k.imag == pytest.approx(4.0 ** liver.eta, rel=1e-12)
    with pytest.raises(ValueError):
        orc.complex_wavenumber(liver, -1.0, 1)
    with pytest.raises(ValueError):
        orc.complex_wavenumber(liver, 1.1e6, 0)


# ------------------------------------------------------------------ grid (test_grid.cpp)
def test_make_grid_covers_and_anchors(orc):  # tests/test_grid.cpp:15-36
    g = orc.make_grid([0, 0, 0], [10e-3, 7e-3, 5e-3], 1e-3, 1)
    assert g.dims == (10, 7, 5) and g.count() == 350
    assert (g.index(1, 0, 0), g.index(0, 1, 0), g.index(0, 0, 1)) == (1, 10, 70)
    anchor = np.array([4.2e-3, 1.3e-3, 2.9e-3])
    ga = orc.make_grid([0, 0, 0], [10e-3, 7e-3, 5e-3], 1e-3, 2, anchor)
    found = any(np.linalg.norm(ga.center(ix, iy, iz) - anchor) < 1e-12
                for iz in range(ga.dims[2]) for iy in range(ga.dims[1]) for ix in range(ga.dims[0]))
    assert found
    assert np.all(ga.lo <= 1e-12) and np.all(ga.hi >= np.array([10e-3, 7e-3, 5e-3]) - 1e-12)


def test_criterion5_golden_mesh_plan(orc):
    # proj/test_output.txt:31 — reference 914x737x737, dx 44.85 um, p2 366x295x295, reduction 15.59
    t = orc.transducer_preset("H131", 100.0, 16)
    plan = orc.plan_nested_meshes(t, water(orc), 10.2e-3, 6, 5)
    assert plan.reference.dims == (914, 737, 737)
    assert f"{plan.reference.dx * 1e6:.4g}" == "44.85"
    assert plan.for_harmonic(2).grid.dims == (366, 295, 295)
    assert f"{plan.reduction_factor(2):.4g}" == "15.59"


def test_nested_plan_invariants(orc):  # tests/test_grid.cpp:52-88
    t = orc.transducer_preset("H131", 100.0, 16)
    w = water(orc)
    d = 10.2e-3
    plan = orc.plan_nested_meshes(t, w, d, 6, 5)
    lam = w.c0 / t.f0
    assert len(plan.grids) == 4
    for n in range(2, 6):
        pg = plan.for_harmonic(n)
        assert pg.grid.dx == pytest.approx(lam / (n * 6), rel=1e-14)
        assert pg.grid.dx * 6 * n * t.f0 / w.c0 == pytest.approx(1.0, rel=1e-12)
        assert pg.domain_hi[0] == pytest.approx(t.focus()[0] + d, rel=1e-12)
        if n > 2:
            prev = plan.for_harmonic(n - 1)
            assert np.all(pg.domain_lo >= prev.domain_lo - 1e-12)
            assert np.all(pg.domain_hi <= prev.domain_hi + 1e-12)
            assert pg.domain_hi[1] - pg.domain_lo[1] == pytest.approx(plan.w * 2.0 / n, rel=1e-12)
            assert plan.for_harmonic(n).grid.count() >= plan.for_harmonic(n - 1).grid.count()
        # focus is a voxel centre of every grid
        g = pg.grid
        i = [round((plan.focus[a] - g.lo[a]) / g.dx - 0.5) for a in range(3)]
        assert np.linalg.norm(g.center(*i) - plan.focus) < 1e-12
    assert plan.reference.dx == pytest.approx(lam / 30, rel=1e-14)
    p2 = orc.plan_nested_meshes(t, w, d, 6, 2)
    assert p2.reduction_factor(2) == pytest.approx(1.0, rel=1e-12)


def _affine(p):
    return complex(2.0 + 100.0 * p[0] - 40.0 * p[1], 7.0 * p[2])


def test_interpolation_constant_and_affine(orc):  # tests/test_grid.cpp:90-122
    coarse = orc.make_grid([0, 0, 0], [8e-3] * 3, 1e-3, 1)
    fine = orc.make_grid([1e-3] * 3, [7e-3] * 3, 0.4e-3, 2)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    f = orc.HarmonicField(coarse, np.full(coarse.count(), 3.0 - 2.0j), k)
    g = orc.interpolate(f, fine)
    assert np.max(np.abs(g.values - (3.0 - 2.0j))) < 1e-14
    vals = np.array([_affine(coarse.center(ix, iy, iz)) for iz in range(coarse.dims[2])
                     for iy in range(coarse.dims[1]) for ix in range(coarse.dims[0])])
    g = orc.interpolate(orc.HarmonicField(coarse, vals, k), fine)
    want = np.array([_affine(fine.center(ix, iy, iz)) for iz in range(fine.dims[2])
                     for iy in range(fine.dims[1]) for ix in range(fine.dims[0])])
    assert np.max(np.abs(g.values - want)) < 1e-12


def test_interpolation_second_order(orc):  # tests/test_grid.cpp:124-157
    target = orc.make_grid([3e-3] * 3, [7e-3] * 3, 0.37e-3, 3)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)

    def gauss(g):
        x, y, z = np.meshgrid(g.centers_axis(0), g.centers_axis(1), g.centers_axis(2), indexing="ij")
        r2 = (x - 5e-3) ** 2 + (y - 5e-3) ** 2 + (z - 5e-3) ** 2
        return np.exp(-r2 / (2 * 2e-3 * 2e-3)).transpose(2, 1, 0).reshape(-1).astype(np.complex128)

    def max_err(h):
        src = orc.make_grid([0, 0, 0], [10e-3] * 3, h, 1)
        out = orc.interpolate(orc.HarmonicField(src, gauss(src), k), target)
        return np.max(np.abs(out.values - gauss(target)))

    r = max_err(1.0e-3) / max_err(0.5e-3)
    assert 3.0 < r < 5.5


def test_interpolation_refuses_far_target(orc):  # tests/test_grid.cpp:159-167
    src = orc.make_grid([0, 0, 0], [4e-3] * 3, 1e-3, 1)
    k = orc.complex_wavenumber(water(orc), 1.1e6, 1)
    f = orc.HarmonicField(src, np.zeros(src.count(), np.complex128), k)
    with pytest.raises(ValueError):
        orc.interpolate(f, orc.make_grid([0, 0, 0], [10e-3, 4e-3, 4e-3], 1e-3, 1))


# ------------------------------------------------------------------ transducer (test_transducer.cpp)
def test_point_layout(orc):  # tests/test_transducer.cpp:50-69
    l, R = 35e-3, 16.5e-3
    cos_tm = math.sqrt(l * l - R * R) / l
    centre = np.array([l, 0, 0])
    for n in (1, 7, 128, 4096):
        pts = orc.distribute_points(l, R, n)
        assert len(pts) == n
        d = np.linalg.norm(pts - centre, axis=1)
        assert np.all(np.abs(d - l) <= 1e-13 * l)
        assert np.all((centre - pts)[:, 0] / l >= cos_tm - 1e-12)
    assert np.linalg.norm(orc.distribute_points(l, R, 1)[0]) == pytest.approx(0.0)
    pts = orc.distribute_points(l, R, 1024)
    dd = np.linalg.norm(pts[:, None, :] - pts[None, :, :], axis=2)
    np.fill_diagonal(dd, np.inf)
    nn = dd.min(axis=1)
    assert nn.max() / nn.min() < 2.0


def _cap_on_axis(l, R, k, x):  # tests/oracles.hpp:22-33
    cos_tm = math.sqrt(l * l - R * R) / l
    z = x - l
    if abs(z) < 1e-9 * l:
        return 0.5 * l * (1.0 - cos_tm) * np.exp(1j * k * l)
    r_pole = abs(z + l)
    r_rim = math.sqrt(z * z + l * l + 2.0 * z * l * cos_tm)
    return (l / (2.0 * z)) * (np.exp(1j * k * r_pole) - np.exp(1j * k * r_rim)) / (1j * k)


def test_monopole_sum_vs_closed_form(orc):  # tests/test_transducer.cpp:71-93
    t = orc.transducer_preset("H131", 100.0, 4096)
    k = orc.complex_wavenumber(water(orc), t.f0, 1)
    xs = [10e-3 + i * (35e-3 / 400.0) for i in range(400)]
    p = orc.unnormalized_field(t, [[x, 0, 0] for x in xs], k)
    exact = np.array([_cap_on_axis(t.focal_length, t.outer_radius, k.k, x) for x in xs])
    assert math.sqrt(np.sum(np.abs(p - exact) ** 2) / np.sum(np.abs(exact) ** 2)) < 0.005


def test_criterion3_on_axis_modulus(orc):  # tests/acceptance.cpp:114-138
    t = orc.transducer_preset("H131", 100.0, 4096)
    k = orc.complex_wavenumber(water(orc), t.f0, 1)
    l, R = t.focal_length, t.outer_radius
    L = math.sqrt(l * l - R * R) - 0.1e-3
    x0, x1 = l - L, l + 10.2e-3
    xs = [x0 + (i + 0.5) * (x1 - x0) / 800 for i in range(800)]
    p = orc.unnormalized_field(t, [[x, 0, 0] for x in xs], k)
    exact = np.abs([_cap_on_axis(l, R, k.k, x) for x in xs])
    rel = 100 * math.sqrt(np.sum((np.abs(p) - exact) ** 2) / np.sum(exact ** 2))
    assert rel < 1.0


def test_power_quadratic_and_target(orc):  # tests/test_transducer.cpp:95-113
    t = orc.transducer_preset("H131", 100.0, 512)
    w = water(orc)
    k = orc.complex_wavenumber(w, t.f0, 1)
    p1 = orc.radiated_power(t, w, k, 1.0, 96, 64)
    p3 = orc.radiated_power(t, w, k, 3.0, 96, 64)
    assert p3 == pytest.approx(9.0 * p1, rel=1e-12) and p1 > 0
    t.power = 40.0
    s = orc.power_scale_factor(t, w, k)
    assert orc.radiated_power(t, w, k, s) == pytest.approx(40.0, rel=1e-12)
    t.power = 0.0
    assert orc.power_scale_factor(t, w, k) == 0.0


def test_monopole_coincidence_throws(orc):  # src/transducer.cpp:112-113
    t = orc.transducer_preset("H131", 100.0, 16)
    k = orc.complex_wavenumber(water(orc), t.f0, 1)
    with pytest.raises(ValueError):
        orc.unnormalized_field(t, [t.source_points[3]], k)


# ------------------------------------------------------------------ cascade (test_cascade.cpp)
def tiny_config(orc, n_harmonics, power, n_w=3):  # tests/test_cascade.cpp:19-27
    w = water(orc)
    t = orc.transducer_preset("H131", power, 128)
    t.f0 = 0.25e6
    plan = orc.plan_nested_meshes(t, w, 6e-3, n_w, n_harmonics, 0.35)
    return orc.CascadeConfig(w, t, plan, n_harmonics)


def test_rhs_coefficients(orc):  # tests/test_cascade.cpp:33-63
    w = water(orc)
    g = orc.make_grid([0, 0, 0], [2e-3] * 3, 1e-3, 1)
    f0 = 1.1e6
    omega = 2 * math.pi * f0
    a, b, c = 2 + 1j, 0.5 - 3j, 1 + 1j
    low = [orc.HarmonicField(g, np.full(g.count(), v), orc.complex_wavenumber(w, f0, i + 1))
           for i, v in enumerate((a, b, c))]
    base = w.beta * omega * omega / (2 * w.rho0 * w.c0 ** 4)
    f2 = orc.rhs_source(2, low[:1], w, omega)
    assert abs(f2[0] - base * 4 * a * a) < 1e-10 * abs(f2[0])
    f3 = orc.rhs_source(3, low[:2], w, omega)
    assert abs(f3[0] - base * 9 * 2 * a * b) < 1e-10 * abs(f3[0])
    f4 = orc.rhs_source(4, low, w, omega)
    assert abs(f4[0] - base * 16 * (b * b + 2 * a * c)) < 1e-10 * abs(f4[0])
    lin = orc.Medium("lin", w.rho0, w.c0, 0.0, w.alpha0, w.eta)
    assert np.max(np.abs(orc.rhs_source(4, low, lin, omega))) == 0.0


def test_cascade_structure_and_homogeneity(orc):  # tests/test_cascade.cpp:65-98
    c1 = tiny_config(orc, 3, 10.0)
    r1 = orc.run_cascade(c1)
    assert len(r1.harmonics) == 3
    assert r1.p(2).grid.dims == c1.plan.for_harmonic(2).grid.dims
    m1, m2, m3 = (np.max(np.abs(r1.p(i).values)) for i in (1, 2, 3))
    assert m3 < m2 < m1 and m3 > 0
    c4 = tiny_config(orc, 3, 40.0)
    r4 = orc.run_cascade(c4)
    for n, s in ((1, 2.0), (2, 4.0), (3, 8.0)):
        a, b = r4.p(n).values, s * r1.p(n).values
        assert np.linalg.norm(a - b) / np.linalg.norm(r1.p(n).values) < 1e-12


def test_cascade_deterministic(orc):  # tests/test_cascade.cpp:100-106
    cfg = tiny_config(orc, 2, 15.0)
    a, b = orc.run_cascade(cfg), orc.run_cascade(cfg)
    assert np.array_equal(a.p(1).values, b.p(1).values)
    assert np.array_equal(a.p(2).values, b.p(2).values)


def test_single_mesh_plan(orc):  # tests/test_cascade.cpp:108-114
    cfg = tiny_config(orc, 3, 10.0)
    single = orc.plan_single_mesh(cfg.transducer, cfg.medium, 6e-3, 3, 3, 0.35)
    assert single.for_harmonic(2).grid.dims == single.reference.dims
    assert single.reduction_factor(2) == pytest.approx(1.0)


# ------------------------------------------------------------------ recorded goldens
@pytest.mark.slow
def test_criterion1_golden_errors(orc):
    # proj/test_output.txt:21 — e(4)=0.6437% e(6)=0.2641% e(8)=0.138% e(10)=0.07983%, slope -2.269
    # tests/acceptance.cpp:47-60: H131 in liver at 30 W, 128 points, focus +-7 lambda x +-1.5 lambda
    liver = orc.medium_preset("liver")
    t = orc.transducer_preset("H131", 30.0, 128)
    lam = liver.c0 / t.f0
    hx, hyz = 7.0 * lam, 1.5 * lam
    fx = t.focus()[0]
    records, slope = orc.quadrature_convergence_study(t, liver, [fx - hx, -hyz, -hyz],
                                                      [fx + hx, hyz, hyz], [4, 6, 8, 10], 20)
    got = {nw: f"{e:.4g}" for nw, e in records}
    assert got == {4: "0.6437", 6: "0.2641", 8: "0.138", 10: "0.07983"}
    assert f"{slope:.4g}" == "-2.269"


def test_direct_potential_at_matches_full_direct_oracle(orc):
    # the sampled-voxel direct sum (used by the full-size GPU checks) is the same formula as
    # direct_potential_oracle (src/potential.cpp:203-238) at every voxel
    g = orc.make_grid([0, 0, 0], [9e-4, 8e-4, 7e-4], 1e-4, 1)
    k = orc.complex_wavenumber(orc.medium_preset("water"), 1.1e6, 1)
    f = orc.random_vector(g.count(), 3)
    full = orc.direct_potential_oracle(k, g, f)
    idx = np.arange(0, g.count(), 7)
    at = orc.direct_potential_at(k, g, f, idx)
    assert np.max(np.abs(at - full[idx])) <= 1e-14 * np.max(np.abs(full))
    with pytest.raises(ValueError):
        orc.direct_potential_at(k, g, f, [g.count()])
