"""BASELINE.json bowl configurations on the reference API (fus mirror or the oracle).

cfg3: uniform-grid 3-harmonic recursion, bowl R=2 cm, l=4 cm, 1 MHz, water (c=1480, rho=1000,
      beta=3.5), surface pressure 0.5 MPa, 4096 points, single mesh bowl face -> 1.2 l, h=lambda3/6.
cfg4: nested 5-harmonic recursion, bowl R=7.5 cm, l=15 cm, 1.1 MHz, c=1540, rho=1050, beta=4.5,
      alpha0=0 (unspecified in BASELINE.json), surface pressure 1 MPa, 4096 points,
      plan_nested_meshes(d=10.2 mm, n_w=6, 5).  `desk=True` scales f0 to 0.275 MHz (same ratios;
      the reference's own tests scale f0 the same way, tests/acceptance.cpp:181).

Surface pressure p0 -> reference amplitude s = 2 Re(k1) p0; run_cascade
always power-normalises (src/cascade.cpp:51-54), so transducer.power = radiated_power(s).
"""
import math


def cfg3(lib, n_points=4096):
    med = lib.Medium("water", 1000.0, 1480.0, 3.5, 0.2, 2.0)
    t = lib.make_bowl("cfg3", 1.0e6, 0.04, 0.02, 0.0, n_points)
    _set_surface_pressure(lib, t, med, 0.5e6)
    plan = lib.plan_single_mesh(t, med, 0.2 * t.focal_length, 6, 3)
    return lib.CascadeConfig(med, t, plan, 3)


def cfg4(lib, desk=True, n_points=4096, n_harmonics=5):
    med = lib.Medium("cfg4", 1050.0, 1540.0, 4.5, 0.0, 1.0)
    f0 = 0.275e6 if desk else 1.1e6
    t = lib.make_bowl("cfg4", f0, 0.15, 0.075, 0.0, n_points)
    _set_surface_pressure(lib, t, med, 1.0e6)
    plan = lib.plan_nested_meshes(t, med, 10.2e-3, 6, n_harmonics)
    return lib.CascadeConfig(med, t, plan, n_harmonics)


def _set_surface_pressure(lib, t, med, p0):
    k1 = lib.complex_wavenumber(med, t.f0, 1)
    s = 2.0 * k1.k.real * p0
    t.power = lib.radiated_power(t, med, k1, s)


def describe(cfg):
    rows = []
    for pg in cfg.plan.grids:
        rows.append((pg.harmonic, tuple(pg.grid.dims), pg.grid.count()))
    return rows
