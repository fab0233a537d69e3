"""Pins of the analysis oracle (oracle/analysis_oracle.py + fus_oracle's on-axis helpers): the
reference's own tests/test_analysis.cpp cases, on CPU."""
import numpy as np
import pytest

from oracle import analysis_oracle as ana
from oracle import fus_oracle as orc

WATER = orc.medium_preset("water")


def test_localisedness_map():  # tests/test_analysis.cpp:79-92
    g = orc.make_grid([0, 0, 0], [3e-3, 1e-3, 1e-3], 1e-3, 1)
    f = orc.HarmonicField(g, np.array([100.0 + 0j, 1j, 0.0]), None)
    q = ana.localisedness_map(f)
    assert q[0] == pytest.approx(0.0) and q[1] == pytest.approx(-2.0)
    assert np.isinf(q[2]) and q[2] < 0


def test_error_trend_diagnostic():  # tests/test_analysis.cpp:94-99
    x = np.array([0.0, 1.0, 2.0])
    p1, p2 = (x, np.full(3, 2.0 + 0j)), (x, np.full(3, 1.0 + 0j))
    assert ana.error_trend_diagnostic(p2, p1, -4.0) == pytest.approx(10.0 * 0.5 * 2.0)
    assert ana.error_trend_diagnostic(p2, p1, 0.0) == pytest.approx(0.0)


def test_shrink_domain_by_threshold():  # src/grid.cpp:114-139
    g = orc.make_grid([0, 0, 0], [5e-3, 4e-3, 3e-3], 1e-3, 1)
    v = np.zeros(g.count(), np.complex128)
    v[g.index(2, 1, 1)] = 10.0
    v[g.index(4, 3, 0)] = 0.05j
    f = orc.HarmonicField(g, v, None)
    lo, hi = ana.shrink_domain_by_threshold(f, 0.0)
    assert np.allclose(lo, [2e-3, 1e-3, 1e-3]) and np.allclose(hi, [3e-3, 2e-3, 2e-3])
    lo, hi = ana.shrink_domain_by_threshold(f, -3.0)
    assert np.allclose(lo, [2e-3, 1e-3, 0.0]) and np.allclose(hi, [5e-3, 4e-3, 2e-3])
    with pytest.raises(ValueError):
        ana.shrink_domain_by_threshold(orc.HarmonicField(g, np.zeros(g.count(), np.complex128), None), -1.0)


def test_quadrature_study_small():  # tests/test_analysis.cpp:101-114
    t = orc.transducer_preset("H131", 20.0, 128)
    t.f0 = 0.25e6
    lam = WATER.c0 / t.f0
    records, slope = orc.quadrature_convergence_study(t, WATER, [35e-3 - lam, -lam / 2, -lam / 2],
                                                      [35e-3 + lam, lam / 2, lam / 2], [2, 3, 4], 8)
    assert len(records) == 3
    assert records[0][1] > records[1][1] > records[2][1]
    assert slope < -1.0


def test_domain_shrink_study_full_level_reproduces_reference():  # tests/test_analysis.cpp:116-131
    t = orc.transducer_preset("H131", 15.0, 128)
    t.f0 = 0.25e6
    plan = ana.plan_full_domain(t, WATER, 6e-3, 3, 2, 0.35)
    cfg = orc.CascadeConfig(WATER, t, plan, 2)
    ref = orc.run_cascade(cfg, workers=8)
    recs = ana.domain_shrink_study(cfg, ref, [1.0, 0.5], False)
    assert len(recs) == 2
    assert recs[0][2] == 1.0 and recs[0][3] < 1e-6
    assert recs[1][3] > recs[0][3] and recs[1][1] == "fraction"
