"""GPU parity of the analysis tooling (src/analysis.cpp): the reference's
recorded acceptance outputs (criterion 1 golden errors and slope, criterion 6 bound), its
tests/test_analysis.cpp cases, and the analysis oracle."""
import time

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
def ana():
    from oracle import analysis_oracle
    return analysis_oracle


def test_criterion1_golden_on_gpu(ctx):
    # proj/test_output.txt:20 (216.88 s in the reference): e(4)=0.6437% e(6)=0.2641% e(8)=0.138%
    # e(10)=0.07983%, slope=-2.269; tests/acceptance.cpp:47-60
    liver = fus.medium_preset("liver")
    t = fus.transducer_preset("H131", 30.0, 128)
    lam = liver.c0 / t.f0
    hx, hyz = 7.0 * lam, 1.5 * lam
    fx = t.focus()[0]
    t0 = time.perf_counter()
    s = fus.quadrature_convergence_study(t, liver, [fx - hx, -hyz, -hyz], [fx + hx, hyz, hyz], [4, 6, 8, 10], 20)
    dt = time.perf_counter() - t0
    got = {int(r.value): f"{r.error_percent:.4g}" for r in s.records}
    assert got == {4: "0.6437", 6: "0.2641", 8: "0.138", 10: "0.07983"}
    assert f"{s.slope:.4g}" == "-2.269"
    print(f"criterion 1 on the GPU: {dt:.2f} s (reference 216.88 s)")


def test_analysis_reference_cases(ctx):  # tests/test_analysis.cpp:26-131
    g = fus.make_grid([0, 0, 0], [3e-3, 1e-3, 1e-3], 1e-3, 1)
    q = fus.localisedness_map(fus.HarmonicField(g, np.array([100.0 + 0j, 1j, 0.0]), None)).cpu().numpy()
    assert q[0] == pytest.approx(0.0) and q[1] == pytest.approx(-2.0) and np.isinf(q[2]) and q[2] < 0
    x = np.array([0.0, 1.0, 2.0])
    ref = fus.OnAxisProfile(x, np.array([1.0, 2.0, 3.0], complex))
    assert fus.on_axis_error(ref, ref, ref) == pytest.approx(0.0)
    zero = fus.OnAxisProfile(x, np.zeros(3, complex))
    assert fus.on_axis_error(zero, ref, ref) == pytest.approx(100.0)
    with pytest.raises(ValueError):
        fus.on_axis_error(ref, ref, zero)
    p1 = fus.OnAxisProfile(x, np.full(3, 2.0 + 0j))
    p2 = fus.OnAxisProfile(x, np.full(3, 1.0 + 0j))
    assert fus.error_trend_diagnostic(p2, p1, -4.0) == pytest.approx(10.0)
    w = fus.medium_preset("water")
    t = fus.transducer_preset("H131", 20.0, 128)
    t.f0 = 0.25e6
    lam = w.c0 / t.f0
    s = fus.quadrature_convergence_study(t, w, [35e-3 - lam, -lam / 2, -lam / 2], [35e-3 + lam, lam / 2, lam / 2],
                                         [2, 3, 4], 8)
    e = [r.error_percent for r in s.records]
    assert e[0] > e[1] > e[2] and s.slope < -1.0


def _shrink_cfg(lib, ana_mod=None):  # tests/test_analysis.cpp:116-124
    w = lib.medium_preset("water")
    t = lib.transducer_preset("H131", 15.0, 128)
    t.f0 = 0.25e6
    plan = (ana_mod or lib).plan_full_domain(t, w, 6e-3, 3, 2, 0.35)
    return lib.CascadeConfig(w, t, plan, 2)


def test_domain_shrink_study_vs_oracle(ctx, orc, ana):
    cfg, cfgo = _shrink_cfg(fus), _shrink_cfg(orc, ana)
    ref, refo = fus.run_cascade(cfg), orc.run_cascade(cfgo, workers=8)
    recs = fus.domain_shrink_study(cfg, ref, [1.0, 0.5], False)
    assert recs[0].value == 1.0 and recs[0].error_percent < 1e-6
    assert recs[1].error_percent > recs[0].error_percent and recs[1].control == "fraction"
    reco = ana.domain_shrink_study(cfgo, refo, [1.0, 0.5], False)
    assert abs(recs[1].error_percent - reco[1][3]) <= 1e-8 * reco[1][3]
    q = fus.domain_shrink_study(cfg, ref, [-1.0, -3.0], True)
    qo = ana.domain_shrink_study(cfgo, refo, [-1.0, -3.0], True)
    for a, b in zip(q, qo):
        assert a.control == "Q0" and abs(a.error_percent - b[3]) <= 1e-8 * b[3] + 1e-12


def test_shrink_box_and_localisedness_vs_oracle(ctx, orc, ana):
    g = fus.make_grid([0, 0, 0], [30e-4, 20e-4, 10e-4], 1e-4, 1)
    rng = np.random.default_rng(3)
    x = np.linspace(-1, 1, g.dims[0])[None, None, :]
    y = np.linspace(-1, 1, g.dims[1])[None, :, None]
    z = np.linspace(-1, 1, g.dims[2])[:, None, None]
    env = np.exp(-8 * (x * x + y * y + z * z)).reshape(-1)
    v = env * (rng.standard_normal(g.count()) + 1j * rng.standard_normal(g.count()))
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 1)
    for q0 in (0.0, -0.5, -2.0, -6.0):
        lo, hi = fus.shrink_domain_by_threshold(fus.HarmonicField(g, v, None), q0)
        loo, hio = ana.shrink_domain_by_threshold(orc.HarmonicField(go, v, None), q0)
        assert np.array_equal(lo, loo) and np.array_equal(hi, hio)
    q = fus.localisedness_map(fus.HarmonicField(g, v, None)).cpu().numpy()
    assert np.allclose(q, ana.localisedness_map(orc.HarmonicField(go, v, None)), rtol=1e-14, atol=1e-14)
    with pytest.raises(ValueError):
        fus.shrink_domain_by_threshold(fus.HarmonicField(g, np.zeros(g.count(), complex), None), -1.0)


def test_criterion6_nested_vs_single_mesh(ctx):
    # tests/acceptance.cpp:175-222 (111.61 s in the reference): each nested harmonic within 1%
    w = fus.medium_preset("water")
    t = fus.transducer_preset("H131", 30.0, 512)
    t.f0 = 0.55e6
    t0 = time.perf_counter()
    single_cfg = fus.CascadeConfig(w, t, fus.plan_single_mesh(t, w, 10.2e-3, 6, 3, 0.5), 3)
    single = fus.run_cascade(single_cfg)
    nested_cfg = fus.CascadeConfig(w, t, fus.plan_nested_meshes(t, w, 10.2e-3, 6, 3, 0.5), 3)
    nested = fus.run_cascade(nested_cfg)
    p1_ref = fus.extract_on_axis(single.p(1))
    errs = []
    for i in (2, 3):
        ref_i = fus.extract_on_axis(single.p(i))
        gi = nested_cfg.plan.for_harmonic(i).grid
        ki = fus.complex_wavenumber(w, t.f0, i)
        lower = [fus.interpolate(nested.p(m), gi) for m in range(1, i)]
        f = fus.rhs_source(i, lower, w, ki.omega)
        nodes = np.stack([ref_i.x, np.zeros_like(ref_i.x), np.zeros_like(ref_i.x)], 1)
        prof = fus.OnAxisProfile(ref_i.x, -fus.evaluate_potential_at(ki, gi, f, nodes), i)
        errs.append(fus.on_axis_error(prof, ref_i, p1_ref))
    dt = time.perf_counter() - t0
    assert all(e < 1.0 for e in errs), errs
    print(f"criterion 6 on the GPU: {dt:.2f} s, err(p2)={errs[0]:.4g}% err(p3)={errs[1]:.4g}% (reference 111.61 s)")
