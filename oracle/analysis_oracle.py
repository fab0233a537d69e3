"""CPU oracle for the analysis tooling: a restatement of the
reference's src/analysis.cpp (localisedness_map, error_trend_diagnostic, plan_full_domain,
domain_shrink_study) and src/grid.cpp:114-139 (shrink_domain_by_threshold), on top of fus_oracle
(extract_on_axis, on_axis_error, quadrature_convergence_study already there). TEST
INFRASTRUCTURE ONLY. Pinned on the reference's tests/test_analysis.cpp cases
(tests/test_oracle_analysis.py). Profiles are (x, p) tuples."""
import math

import numpy as np

from oracle import fus_oracle as orc


def localisedness_map(fld: orc.HarmonicField) -> np.ndarray:
    """src/analysis.cpp:80-90: log10(|f| / max|f|), -inf for zero voxels."""
    a = np.abs(fld.values)
    m = float(a.max()) if a.size else 0.0
    if m <= 0.0:
        raise ValueError("localisedness_map: field is identically zero")
    q = np.full(a.size, -np.inf)
    nz = a > 0.0
    q[nz] = np.log10(a[nz] / m)
    return q


def shrink_domain_by_threshold(fld: orc.HarmonicField, q0: float):
    """src/grid.cpp:114-139 -> (lo, hi) of the tightest box holding |f| >= max 10^q0."""
    g = fld.grid
    a = np.abs(fld.values)
    m = float(a.max())
    if m <= 0.0:
        raise ValueError("shrink_domain_by_threshold: field is identically zero")
    thr = m if q0 >= 0.0 else m * math.pow(10.0, q0)
    idx = np.nonzero(a >= thr)[0]
    ix, iy, iz = idx % g.dims[0], (idx // g.dims[0]) % g.dims[1], idx // (g.dims[0] * g.dims[1])
    lo_i = np.array([ix.min(), iy.min(), iz.min()])
    hi_i = np.array([ix.max(), iy.max(), iz.max()])
    return g.lo + lo_i * g.dx, g.lo + (hi_i + 1) * g.dx


def error_trend_diagnostic(p_i, p1, q0: float) -> float:
    """src/analysis.cpp:243-246"""
    on_p1 = orc._resample(p_i[0], p_i[1], p1[0])
    return 10.0 * (np.linalg.norm(on_p1) / np.linalg.norm(p1[1])) * math.sqrt(abs(q0))


def plan_full_domain(t, m, d, n_w, n_harmonics, width_scale=1.0) -> orc.MeshPlan:
    """src/analysis.cpp:164-174: every harmonic keeps the D_2 domain at its own resolution."""
    plan = orc.plan_nested_meshes(t, m, d, n_w, n_harmonics, width_scale)
    d2lo, d2hi = plan.grids[0].domain_lo.copy(), plan.grids[0].domain_hi.copy()
    lambda1 = m.c0 / t.f0
    for pg in plan.grids:
        pg.domain_lo, pg.domain_hi = d2lo.copy(), d2hi.copy()
        pg.grid = orc.make_grid(d2lo, d2hi, lambda1 / (pg.harmonic * n_w), pg.harmonic, plan.focus)
    return plan


def domain_shrink_study(cfg, reference, levels, q0_mode: bool):
    """src/analysis.cpp:176-241 -> [(harmonic, control, level, error %)]"""
    medium, t, plan = cfg.medium, cfg.transducer, cfg.plan
    lambda1 = medium.c0 / t.f0
    focus = plan.focus
    p1_ref = orc.extract_on_axis(reference.p(1))
    records = []
    for i in range(2, cfg.n_harmonics + 1):
        pi_ref = orc.extract_on_axis(reference.p(i))
        full = plan.for_harmonic(i)
        ki = orc.complex_wavenumber(medium, t.f0, i)
        integrand = None
        if q0_mode:
            lower = [reference.p(mm) if orc.same_grid(reference.p(mm).grid, full.grid)
                     else orc.interpolate(reference.p(mm), full.grid) for mm in range(1, i)]
            integrand = orc.HarmonicField(full.grid, orc.rhs_source(i, lower, medium, ki.omega), ki)
        for level in levels:
            if q0_mode:
                lo, hi = shrink_domain_by_threshold(integrand, level)
            else:
                L = focus[0] - full.domain_lo[0]
                w = full.domain_hi[1]
                lo = np.array([focus[0] - level * L, -level * w, -level * w])
                hi = np.array([full.domain_hi[0], level * w, level * w])
            grid = orc.make_grid(lo, hi, lambda1 / (i * plan.n_w), i, focus)
            lower = [orc.interpolate(reference.p(mm), grid) for mm in range(1, i)]
            f = orc.rhs_source(i, lower, medium, ki.omega)
            nodes = np.stack([pi_ref[0], np.zeros_like(pi_ref[0]), np.zeros_like(pi_ref[0])], 1)
            prof = (pi_ref[0], -orc.evaluate_potential_at(ki, grid, f, nodes))
            records.append((i, "Q0" if q0_mode else "fraction", float(level),
                            orc.on_axis_error(prof, pi_ref, p1_ref)))
    return records
