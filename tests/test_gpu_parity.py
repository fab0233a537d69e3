"""GPU parity: the CUDA path (through the C-ABI) against the pinned CPU oracle.

Tolerances: the reference's own (1e-12 / 1e-13 for the FFT-free known-answer tests) and
north_star's relative L2 <= 1e-10 per complex128 field; integer/index work (grids, crop,
interpolation, rhs) must be bit-exact.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2011_03009_b200 import fus  # noqa: E402


def rel_l2(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = b.cpu().numpy() if hasattr(b, "cpu") else np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def host(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def ctx():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return fus.context(0)


def water():
    return fus.medium_preset("water")


# ------------------------------------------------------------------ volume potential KATs
@pytest.mark.parametrize("seed,pad", [(1234, False), (1234, True), (2024, False)])
def test_apply_matches_direct_20x18x16(ctx, orc, seed, pad):
    # tests/test_potential.cpp:75-92, tests/acceptance.cpp:98-112 (< 1e-12 rel max-norm)
    g = fus.make_grid([0, 0, 0], [20e-4, 18e-4, 16e-4], 1e-4, 2)
    assert g.dims == (20, 18, 16)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), seed)
    u = host(fus.GreenKernel(g, k, pad).apply(f))
    go = orc.make_grid([0, 0, 0], [20e-4, 18e-4, 16e-4], 1e-4, 2)
    ref = orc.direct_potential_oracle(orc.complex_wavenumber(orc.medium_preset("water"), 1.1e6, 2), go, f)
    assert np.max(np.abs(u - ref)) < 1e-12 * np.max(np.abs(ref))


def test_delta_reproduces_kernel_column(ctx):
    # tests/test_potential.cpp:117-139 (1e-13 rel + 1e-20 abs; exact crop and indexing)
    g = fus.make_grid([0, 0, 0], [9e-4, 8e-4, 7e-4], 1e-4, 1)
    k = fus.complex_wavenumber(water(), 1.1e6, 1)
    delta = np.zeros(g.count(), np.complex128)
    j = g.index(4, 3, 2)
    delta[j] = 1.0
    col = host(fus.GreenKernel(g, k).apply(delta))
    vol = g.dx ** 3
    xj = g.center(4, 3, 2)
    for iz in range(g.dims[2]):
        for iy in range(g.dims[1]):
            for ix in range(g.dims[0]):
                i = g.index(ix, iy, iz)
                want = fus.self_weight(k, g.dx) if i == j else vol * fus.green_function(g.center(ix, iy, iz), xj, k)
                assert abs(col[i] - want) < 1e-13 * abs(want) + 1e-20


def test_apply_linear_and_translation_covariant(ctx):
    # tests/test_potential.cpp:94-115
    g = fus.make_grid([-3e-3, 1e-3, 0], [2e-3, 6e-3, 4e-3], 5e-4, 1)
    k = fus.complex_wavenumber(water(), 1.1e6, 1)
    K = fus.GreenKernel(g, k)
    f, h = fus.random_vector(g.count(), 7), fus.random_vector(g.count(), 8)
    a = complex(0.3, -1.7)
    lhs = host(K.apply(a * f + h))
    rhs = a * host(K.apply(f)) + host(K.apply(h))
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(rhs))
    off = np.array([11e-3, -4e-3, 9e-3])
    K2 = fus.GreenKernel(fus.VoxelGrid(g.lo + off, g.hi + off, g.dx, g.dims, 1), k)
    u = host(K.apply(f))
    assert np.max(np.abs(host(K2.apply(f)) - u)) < 1e-12 * np.max(np.abs(u))


@pytest.mark.parametrize("dims", [(1, 1, 1), (1, 5, 3), (7, 6, 5), (13, 11, 2), (33, 1, 9),
                                  (16, 16, 16), (25, 30, 7), (64, 3, 40),
                                  # Pz = 256 / 512 with pruned halves: the two-stage pass C
                                  # (odd line count 9 x 5 exercises the half-filled last pair)
                                  (9, 7, 128), (5, 3, 256), (3, 2, 100), (6, 5, 129), (4, 3, 200),
                                  # Nz = 300 / 341: Pz = 768 (multi-warp pass C) instead of 600 / 686
                                  (3, 2, 300), (2, 3, 341),
                                  # Nz = 490: Pz = 1024 (two-warp-line pass C)
                                  (2, 2, 490),
                                  # Pz = 768 (3 x 256 half-warp pass C) with an odd line count
                                  # (the last CTA pair holds one line), Pz = 1024 with odd lines
                                  (5, 3, 333), (3, 3, 300), (5, 3, 500),
                                  # Nz = 768 / 1024: Pz = 1536 / 2048 (two- / four-warp lines)
                                  (3, 2, 768), (2, 3, 1024),
                                  # Nz = 600 / 900: Pz = 1536 / 2048 preferred over 1200 / 1800
                                  (2, 2, 600), (2, 1, 900),
                                  # Nx / Ny = 512, 768, 1024: Px / Py = 1024, 1536, 2048 (multi-
                                  # warp-line transposing passes; ragged T-line tiles)
                                  (512, 5, 3), (3, 512, 4), (768, 3, 2), (2, 768, 3),
                                  # Px / Py / Pz = 1536 = 3 x 512 kernels with fewer valid
                                  # positions and ragged 4-line tiles
                                  (700, 5, 3), (3, 650, 5), (601, 7, 2), (6, 5, 700), (9, 2, 601),
                                  (1024, 2, 2), (2, 1024, 2),
                                  # Nx / Ny in (128, 256]: Px / Py = 512 (16x16x2 transposing passes)
                                  (200, 3, 2), (3, 230, 4), (256, 7, 3),
                                  # Px = Py = 512: passes A+B fused through the z-slab ring
                                  # (slabs of 8 planes, ragged last slab, single slab)
                                  (200, 150, 13), (130, 129, 37), (256, 256, 3)])
def test_apply_ragged_sizes_vs_oracle(ctx, orc, dims):
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    assert g.dims == dims
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), 99)
    u = host(fus.GreenKernel(g, k).apply(f))
    go = orc.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    ko = orc.complex_wavenumber(orc.medium_preset("water"), 1.1e6, 2)
    ref = orc.GreenKernel(go, ko).apply(f)
    assert rel_l2(u, ref) <= 1e-12
    if g.count() <= 4000:
        d = orc.direct_potential_oracle(ko, go, f)
        assert np.max(np.abs(u - d)) < 1e-12 * np.max(np.abs(d))


def cfg1_grid():
    c, f = 1540.0, 1.1e6
    h = (c / f) / 6.0
    return fus.make_grid([0, 0, 0], [64 * h, 64 * h, 64 * h], h, 1), fus.Wavenumber(
        complex(2 * math.pi * f / c, 0.0), 1, 2 * math.pi * f)


def test_config1_64cubed_vs_oracle(ctx, orc):
    # BASELINE config 1: 64^3, h = lambda/6 at 1.1 MHz, c = 1540, iid U[-1,1] seed 1234
    g, k = cfg1_grid()
    assert g.dims == (64, 64, 64)
    f = fus.random_vector(g.count(), 1234)
    K = fus.GreenKernel(g, k)
    assert K.padded == (128, 128, 128)
    u = K.apply(f)
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 1)
    ref = orc.GreenKernel(go, orc.Wavenumber(k.k, 1, k.omega), workers=8).apply(f)
    assert rel_l2(u, ref) <= 1e-10
    # host-vector drop-in gives the same bits as the device apply
    assert np.array_equal(K.apply_host(f), host(u))
    # scale argument: -apply
    assert np.array_equal(host(K.apply(f, -1.0)), -host(u))


def cfg2_source(g, seed=2024):
    f = fus.random_vector(g.count(), seed).reshape(g.dims[2], g.dims[1], g.dims[0])
    c = 0.5 * (g.lo + g.hi)
    sig = 0.2 * (g.hi[0] - g.lo[0])
    x = g.lo[0] + (np.arange(g.dims[0]) + 0.5) * g.dx
    y = g.lo[1] + (np.arange(g.dims[1]) + 0.5) * g.dx
    z = g.lo[2] + (np.arange(g.dims[2]) + 0.5) * g.dx
    r2 = ((x - c[0]) ** 2)[None, None, :] + ((y - c[1]) ** 2)[None, :, None] + ((z - c[2]) ** 2)[:, None, None]
    return (f * np.exp(-r2 / (2 * sig * sig))).reshape(-1)


def cfg2_grid():
    c, f0 = 1540.0, 1.1e6
    k2 = 2 * 2 * math.pi * f0 / c
    h = (c / (2 * f0)) / 6.0
    return fus.make_grid([0, 0, 0], [256 * h] * 3, h, 2), fus.Wavenumber(complex(k2, 0.0), 2, 2 * math.pi * f0)


def test_config2_256cubed_vs_oracle(ctx, orc):
    g, k = cfg2_grid()
    assert g.dims == (256, 256, 256)
    f = cfg2_source(g)
    K = fus.GreenKernel(g, k)
    assert K.padded == (512, 512, 512)
    u = K.apply(f)
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 2)
    ref = orc.GreenKernel(go, orc.Wavenumber(k.k, 2, k.omega), workers=16).apply(f)
    assert rel_l2(u, ref) <= 1e-10
    # host-vector apply (default: 8 z-chunks pipelined against the copies) gives the same bits
    assert np.array_equal(K.apply_host(f), host(u))


@pytest.mark.parametrize("dims", [(25, 30, 7), (33, 1, 9), (16, 16, 16), (64, 3, 40)])
@pytest.mark.parametrize("chunks", ["1", "2", "3", "7", "64"])
def test_host_apply_chunk_pipeline_is_bitwise_device_apply(ctx, monkeypatch, dims, chunks):
    # the z-chunked host pipeline (H2D | passes A+B per chunk, pass C, passes D+E | D2H per
    # chunk) splits no line, so ragged chunkings must reproduce the one-shot apply exactly
    monkeypatch.setenv("FUSG_HOST_CHUNKS", chunks)
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    K = fus.GreenKernel(g, fus.complex_wavenumber(water(), 1.1e6, 2))
    f = fus.random_vector(g.count(), 5)
    want = host(K.apply(f, 0.5))
    for _ in range(2):  # back-to-back calls reuse the staging buffers and events
        assert np.array_equal(K.apply_host(f, 0.5), want)


# ------------------------------------------------------------------ off-grid potential (8(f) rank 1)
@pytest.mark.parametrize("att", [True, False])
def test_evaluate_potential_at_vs_oracle(ctx, orc, att):
    # src/potential.cpp:161-201: on-grid points (self term), off-grid points, points outside the
    # box, zero-f voxels (skipped); attenuating water or real k
    g = fus.make_grid([0, 0, 0], [23e-4, 19e-4, 17e-4], 1e-4, 2)
    go = orc.make_grid([0, 0, 0], [23e-4, 19e-4, 17e-4], 1e-4, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    if not att:
        k = fus.Wavenumber(complex(k.k.real, 0.0), 2, k.omega)
    ko = orc.Wavenumber(k.k, 2, k.omega)
    f = fus.random_vector(g.count(), 21)
    f[::7] = 0.0
    rng = np.random.default_rng(5)
    pts = [g.center(ix, iy, iz) for ix, iy, iz in ((0, 0, 0), (5, 7, 3), (22, 18, 16))]
    pts += list(g.lo + rng.random((40, 3)) * (g.hi - g.lo))
    pts += [g.hi + np.array([3e-3, -1e-3, 2e-3]), g.lo - np.array([1e-2, 0, 0])]
    got = fus.evaluate_potential_at(k, g, f, pts)
    ref = orc.evaluate_potential_at(ko, go, f, pts)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    # deterministic
    assert np.array_equal(fus.evaluate_potential_at(k, g, torch.from_numpy(f).cuda(), pts), got)
    with pytest.raises(ValueError):
        fus.evaluate_potential_at(k, g, f[:5], pts)


def test_evaluate_potential_at_agrees_with_apply_at_centres(ctx):
    # tests/test_potential.cpp:181-207 (1e-12 of max |u|), on a 64^3 grid with 4096 points
    g = fus.make_grid([0, 0, 0], [64e-4] * 3, 1e-4, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), 99)
    u = host(fus.GreenKernel(g, k).apply(f))
    rng = np.random.default_rng(1)
    ii = rng.integers(0, 64, (4096, 3))
    pts = [g.center(*t) for t in ii]
    v = fus.evaluate_potential_at(k, g, f, pts)
    idx = [g.index(*t) for t in ii]
    assert np.max(np.abs(v - u[idx])) < 1e-12 * np.max(np.abs(u))


# ------------------------------------------------------------------ incident field
def test_monopole_grid_and_points_vs_oracle(ctx, orc):
    t = fus.transducer_preset("H131", 100.0, 4096)
    to = orc.transducer_preset("H131", 100.0, 4096)
    w, wo = water(), orc.medium_preset("water")
    plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 2, 0.3)
    g = plan.for_harmonic(2).grid
    p = fus.evaluate_first_harmonic(t, w, g, 3.0)
    go = orc.VoxelGrid(g.lo, g.hi, g.dx, g.dims, 2)
    ref = orc.evaluate_first_harmonic(to, wo, go, 3.0).values
    assert rel_l2(p.values, ref) <= 1e-12
    k = fus.complex_wavenumber(w, t.f0, 1)
    xs = [[10e-3 + i * (35e-3 / 400.0), 0, 0] for i in range(400)]
    pp = fus.unnormalized_field(t, xs, k)
    ref = orc.unnormalized_field(to, xs, orc.complex_wavenumber(wo, to.f0, 1))
    assert rel_l2(pp, ref) <= 1e-12


def test_monopole_coincidence_raises(ctx):
    t = fus.transducer_preset("H131", 100.0, 16)
    k = fus.complex_wavenumber(water(), t.f0, 1)
    with pytest.raises(ValueError):
        fus.unnormalized_field(t, [t.source_points[3]], k)
    # the context stays usable afterwards
    assert fus.unnormalized_field(t, [[20e-3, 0, 0]], k).shape[0] == 1


def test_radiated_power_vs_oracle(ctx, orc):
    t = fus.transducer_preset("H131", 40.0, 512)
    to = orc.transducer_preset("H131", 40.0, 512)
    w, wo = water(), orc.medium_preset("water")
    k, ko = fus.complex_wavenumber(w, t.f0, 1), orc.complex_wavenumber(wo, to.f0, 1)
    for (nr, nt) in ((96, 64), (384, 256)):
        a = fus.radiated_power(t, w, k, 1.0, nr, nt)
        b = orc.radiated_power(to, wo, ko, 1.0, nr, nt)
        assert abs(a - b) <= 1e-12 * abs(b)
    s = fus.power_scale_factor(t, w, k)
    assert fus.radiated_power(t, w, k, s) == pytest.approx(40.0, rel=1e-12)
    # deterministic: identical bits on repeat
    assert fus.radiated_power(t, w, k, 1.0) == fus.radiated_power(t, w, k, 1.0)


# ------------------------------------------------------------------ transfer + source (bit-exact)
def test_interpolate_bit_exact(ctx, orc):
    w = water()
    k = fus.complex_wavenumber(w, 1.1e6, 1)
    src = fus.make_grid([0, 0, 0], [8e-3] * 3, 1e-3, 1)
    for tgt in (fus.make_grid([1e-3] * 3, [7e-3] * 3, 0.4e-3, 2),
                fus.make_grid([-0.5e-3] * 3, [8.5e-3] * 3, 0.37e-3, 3),
                fus.make_grid([0, 0, 0], [8e-3, 8e-3, 1e-3], 1e-3, 1)):
        f = fus.random_vector(src.count(), 5)
        out = fus.interpolate(fus.HarmonicField(src, f, k), tgt)
        so = orc.VoxelGrid(src.lo, src.hi, src.dx, src.dims)
        to = orc.VoxelGrid(tgt.lo, tgt.hi, tgt.dx, tgt.dims)
        ref = orc.interpolate(orc.HarmonicField(so, f, None), to).values
        assert np.array_equal(host(out.values), ref)
    with pytest.raises(ValueError):
        fus.interpolate(fus.HarmonicField(src, fus.random_vector(src.count(), 1), k),
                        fus.make_grid([0, 0, 0], [20e-3, 8e-3, 8e-3], 1e-3, 1))


def test_rhs_source_bit_exact(ctx, orc):
    w, wo = water(), orc.medium_preset("water")
    g = fus.make_grid([0, 0, 0], [10e-3, 7e-3, 5e-3], 1e-3, 1)
    omega = 2 * math.pi * 1.1e6
    fields = [fus.random_vector(g.count(), 10 + i) for i in range(5)]
    for n in (2, 3, 4, 6):
        lower = [fus.HarmonicField(g, fields[i], None) for i in range(n - 1)]
        got = host(fus.rhs_source(n, lower, w, omega))
        lo = [orc.HarmonicField(None, fields[i], None) for i in range(n - 1)]
        assert np.array_equal(got, orc.rhs_source(n, lo, wo, omega))
    with pytest.raises(ValueError):
        fus.rhs_source(1, [], w, omega)


@pytest.mark.gpu
def test_rhs_source_full_conjugate_terms(ctx, orc):
    """Eq. (cascade_1) with the p_m conj(p_{m-n}) terms (north_star (2)); M = n - 1 is rhs_source."""
    w, wo = water(), orc.medium_preset("water")
    g = fus.make_grid([0, 0, 0], [10e-3, 7e-3, 5e-3], 1e-3, 1)
    omega = 2 * math.pi * 1.1e6
    fields = [fus.random_vector(g.count(), 40 + i) for i in range(6)]
    hf = [fus.HarmonicField(g, v, None) for v in fields]
    ho = [orc.HarmonicField(None, v, None) for v in fields]
    for n in (2, 3, 4):
        assert np.array_equal(host(fus.rhs_source_full(n, hf[: n - 1], w, omega)),
                              host(fus.rhs_source(n, hf[: n - 1], w, omega)))
        for M in range(n, 7):
            got = host(fus.rhs_source_full(n, hf[:M], w, omega))
            assert np.array_equal(got, orc.rhs_source_full(n, ho[:M], wo, omega)), (n, M)
    # p_n enters only through p_{2n} conj(p_n): with 2n > M its slot may be None
    withnone = list(hf[:5])
    withnone[2] = None
    assert np.array_equal(host(fus.rhs_source_full(3, withnone, w, omega)),
                          host(fus.rhs_source_full(3, hf[:5], w, omega)))
    withnone = list(hf[:4])
    withnone[1] = None
    with pytest.raises(ValueError):  # n = 2, M = 4: p_4 conj(p_2) needs p_2
        fus.rhs_source_full(2, withnone, w, omega)
    with pytest.raises(ValueError):
        fus.rhs_source_full(4, hf[:2], w, omega)


# ------------------------------------------------------------------ recursion
def tiny(n_h, power, lib):
    w = lib.medium_preset("water")
    t = lib.transducer_preset("H131", power, 128)
    t.f0 = 0.25e6
    return lib.CascadeConfig(w, t, lib.plan_nested_meshes(t, w, 6e-3, 3, n_h, 0.35), n_h)


def test_cascade_vs_oracle_tiny(ctx, orc):
    # tests/test_cascade.cpp:19-27 tiny_config, 3 harmonics: each field <= 1e-10 rel L2
    r = fus.run_cascade(tiny(3, 20.0, fus))
    ro = orc.run_cascade(tiny(3, 20.0, orc))
    assert len(r.harmonics) == 3 and len(r.timings) == 2
    for n in (1, 2, 3):
        assert r.p(n).grid.dims == ro.p(n).grid.dims
        assert rel_l2(r.p(n).values, ro.p(n).values) <= 1e-10, n
    assert r.source_normalization == pytest.approx(ro.source_normalization, rel=1e-12)
    assert [t.harmonic for t in r.timings] == [2, 3]
    assert r.timings[0].voxels == r.p(2).grid.count()


def test_cascade_homogeneity_and_determinism(ctx):
    # tests/test_cascade.cpp:84-106 and acceptance criterion 7
    r1 = fus.run_cascade(tiny(3, 10.0, fus))
    r4 = fus.run_cascade(tiny(3, 40.0, fus))
    for n, s in ((1, 2.0), (2, 4.0), (3, 8.0)):
        a, b = host(r4.p(n).values), s * host(r1.p(n).values)
        assert np.linalg.norm(a - b) / np.linalg.norm(host(r1.p(n).values)) < 1e-12
    again = fus.run_cascade(tiny(3, 10.0, fus))
    for n in (1, 2, 3):
        assert torch.equal(again.p(n).values, r1.p(n).values)


def test_cascade_recompute_p1_and_single_mesh(ctx, orc):
    cfg, cfgo = tiny(3, 20.0, fus), tiny(3, 20.0, orc)
    cfg.recompute_p1_each_grid = cfgo.recompute_p1_each_grid = True
    r, ro = fus.run_cascade(cfg), orc.run_cascade(cfgo)
    for n in (1, 2, 3):
        assert rel_l2(r.p(n).values, ro.p(n).values) <= 1e-10
    t, to = cfg.transducer, cfgo.transducer
    cfg.plan = fus.plan_single_mesh(t, cfg.medium, 6e-3, 3, 3, 0.35)
    cfgo.plan = orc.plan_single_mesh(to, cfgo.medium, 6e-3, 3, 3, 0.35)
    r, ro = fus.run_cascade(cfg), orc.run_cascade(cfgo)
    for n in (1, 2, 3):
        assert rel_l2(r.p(n).values, ro.p(n).values) <= 1e-10


def test_launch_counter_counts_library_kernels(ctx):
    g, k = cfg1_grid()
    K = fus.GreenKernel(g, k)
    before = ctx.launch_count()
    K.apply(fus.random_vector(g.count(), 3))
    assert ctx.launch_count() - before == 5  # passes A..E


def _reduced_cfg4(lib):
    # BASELINE config 4 geometry (bowl R 7.5 cm, l 15 cm, c 1540, rho 1050, beta 4.5, 1 MPa
    # surface pressure, nested plan d=10.2 mm, n_w=6, 5 harmonics) at f0 = 1.1 MHz / 8 with
    # 256 points so the CPU oracle finishes in seconds (the reference's own tests scale f0 the
    # same way, tests/acceptance.cpp:181).
    med = lib.Medium("cfg4", 1050.0, 1540.0, 4.5, 0.0, 1.0)
    t = lib.make_bowl("cfg4", 1.1e6 / 8, 0.15, 0.075, 0.0, 256)
    k1 = lib.complex_wavenumber(med, t.f0, 1)
    return med, t, k1


def test_nested_5_harmonic_cascade_vs_oracle(ctx, orc):
    med, t, k1 = _reduced_cfg4(fus)
    medo, to, k1o = _reduced_cfg4(orc)
    s = 2.0 * k1.k.real * 1.0e6  # surface pressure -> amplitude
    t.power = fus.radiated_power(t, med, k1, s)
    to.power = orc.radiated_power(to, medo, k1o, s)
    assert t.power == pytest.approx(to.power, rel=1e-12)
    cfg = fus.CascadeConfig(med, t, fus.plan_nested_meshes(t, med, 10.2e-3, 6, 5), 5)
    cfgo = orc.CascadeConfig(medo, to, orc.plan_nested_meshes(to, medo, 10.2e-3, 6, 5), 5)
    r = fus.run_cascade(cfg)
    ro = orc.run_cascade(cfgo, workers=16)
    assert r.source_normalization == pytest.approx(s, rel=1e-9)
    for n in range(1, 6):
        assert r.p(n).grid.dims == ro.p(n).grid.dims
        assert rel_l2(r.p(n).values, ro.p(n).values) <= 1e-10, n
    assert [row.harmonic for row in r.timings] == [2, 3, 4, 5]


def test_cpp_dropin_api_all_cases(ctx):
    """C++ namespace-fus drop-in: host + device cases (apply vs direct quadrature, delta
    column, rhs, interpolation, power normalisation, cascade homogeneity/determinism)."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "test_fus_api")
    out = subprocess.run([exe, "all"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.parametrize("dims,applies", [((106, 105, 105), 40), ((130, 105, 127), 40), ((256, 256, 256), 12),
                                          ((64, 64, 700), 12), ((100, 100, 380), 12), ((200, 200, 490), 6),
                                          # the TMA-tiled transposing passes at 1536 and 1024 (x and y)
                                          ((768, 64, 20), 10), ((64, 768, 20), 10), ((500, 37, 9), 20),
                                          ((9, 500, 37), 20)])
def test_repeated_applies_are_bitwise_identical(ctx, dims, applies):
    # Every staged pass C (L = 256 / 512 / 1536 / 768 / 1024) refills its shared buffers with bulk
    # copies while other lanes have just read them; without the async-proxy fence the refill
    # occasionally overtook a queued shared load (about one apply in ten at 224 x 224 lines of
    # L = 256 differed, up to 0.7 % in max norm). Repeated applies must agree bit for bit.
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 4)
    k = fus.complex_wavenumber(water(), 0.8e6, 4)
    f = torch.from_numpy(fus.random_vector(g.count(), 4)).cuda()
    K = fus.GreenKernel(g, k)
    ref = K.apply(f)
    for _ in range(applies):
        assert torch.equal(K.apply(f), ref)


@pytest.mark.parametrize("dims,G", [((37, 20, 19), 2), ((37, 20, 19), 3), ((64, 64, 64), 4),
                                    ((16, 24, 9), 8), ((25, 30, 7), 7),
                                    # Pz = 512: the 16x16x2 pass C on kx slabs (kx offset, no mirror order)
                                    ((37, 20, 150), 2), ((37, 20, 150), 3)])
def test_slab_sharded_apply_loopback_is_bitwise_unsharded(ctx, dims, G):
    # the sharded apply uses the same pass kernels and differs only in data
    # movement, so every decomposition must reproduce the single-GPU apply bit for bit.
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), 5)
    want = fus.GreenKernel(g, k).apply(f)
    got = fus.apply_slab_loopback(g, k, f, G)
    assert torch.equal(got, want)


@pytest.mark.parametrize("dims,G", [((128, 128, 19), 2), ((128, 126, 19), 3), ((256, 255, 9), 4),
                                    ((128, 128, 40), 8), ((127, 128, 23), 7),
                                    # Px = 1536 / Py = 1024: the multi-warp-line transposing kernels
                                    ((768, 512, 5), 3)])
def test_slab_fused_peer_transposes_loopback_is_bitwise_unsharded(ctx, dims, G):
    # The transposes fused into passes A and D (peer stores, no exchange buffers): every rank's
    # pass A writes each kx segment into the owner's x-slab, pass D each z-row into the owner's
    # A slab; ragged z and kx splits; must reproduce the single-GPU apply bit for bit.
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    assert fus.padded_dims(g)[0] in (256, 512, 1536) and fus.padded_dims(g)[1] in (256, 512, 1024)
    f = fus.random_vector(g.count(), 9)
    want = fus.GreenKernel(g, k).apply(f, 0.5)
    got = fus.apply_slab_loopback(g, k, f, G, 0.5, transport="p2p")
    assert torch.equal(got, want)


@pytest.mark.parametrize("dims,G", [((37, 20, 19), 2), ((64, 64, 64), 4), ((25, 30, 7), 7), ((128, 128, 40), 8)])
def test_slab_kernels_hold_only_their_octant_rows(ctx, dims, G):
    # SURVEY.md 8(e) "octant kept per x-slab": rank r keeps the folded kx rows of its columns
    # [x0, x0 + nx) (built without a collective); together the ranks cover the whole octant,
    # each holds about 2/G of it, and the applies above stay bitwise the unsharded ones.
    dx = 1e-4
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    Px = fus.padded_dims(g)[0]
    Hx = Px // 2 + 1
    full = fus.GreenKernel(g, k)
    covered = set()
    for r in range(G):
        sk = fus.SlabKernel(g, k, G, r)
        kf0, knf = sk.octant_rows
        folds = {min(x, Px - x) for x in range(sk.x0, sk.x0 + sk.nx)}
        assert folds == set(range(kf0, kf0 + knf)), (r, kf0, knf)
        assert knf <= sk.nx and (G < 4 or knf < Hx)
        covered |= folds
    assert covered == set(range(Hx))
    f = fus.random_vector(g.count(), 17)
    assert torch.equal(fus.apply_slab_loopback(g, k, f, G), full.apply(f))


def test_slab_fused_transposes_need_warp_lengths(ctx):
    g = fus.make_grid([0, 0, 0], [37e-4, 20e-4, 19e-4], 1e-4, 2)  # Px = 80: no transposing warp kernel
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    with pytest.raises(ValueError, match="fused transposes need a padded x length"):
        fus.apply_slab_loopback(g, k, fus.random_vector(g.count(), 1), 2, transport="p2p")


def test_slab_fused_p2p_over_nccl_single_rank_with_ipc_handles(ctx):
    # The multi-process entry points on one rank: IPC handle export, peer attach (own buffers),
    # the fused apply with its NCCL stream barriers; bitwise = unsharded.
    g = fus.make_grid([0, 0, 0], [128e-4, 128e-4, 21e-4], 1e-4, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), 13)
    want = fus.GreenKernel(g, k).apply(f)
    c = fus.Context(0)
    fus.attach_nccl(c, 1, 0, fus.nccl_unique_id())
    sk = fus.SlabKernel(g, k, 1, 0, c)
    with pytest.raises(ValueError, match="peers not attached"):
        sk.apply_p2p(torch.from_numpy(f).cuda())
    h = sk.ipc_handles()
    assert len(h) == 128
    sk.attach_peers(h)
    for _ in range(2):
        assert torch.equal(sk.apply_p2p(torch.from_numpy(f).cuda()), want)


def test_slab_apply_over_nccl_single_rank(ctx):
    # The NCCL transport's full path (phase A, grouped send/recv, unpack, B-D, pack, send/recv,
    # phase E) on a 1-rank communicator: every NCCL call runs (to self); bitwise = unsharded.
    g = fus.make_grid([0, 0, 0], [37e-4, 20e-4, 19e-4], 1e-4, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    f = fus.random_vector(g.count(), 11)
    want = fus.GreenKernel(g, k).apply(f)
    c = fus.Context(0)
    fus.attach_nccl(c, 1, 0, fus.nccl_unique_id())
    sk = fus.SlabKernel(g, k, 1, 0, c)
    got = sk.apply(torch.from_numpy(f).cuda())
    assert torch.equal(got, want)
    # and the loopback transport with G = 1 takes the same exchange path
    assert torch.equal(fus.apply_slab_loopback(g, k, f, 1, ctx=c), want)


_AB_FUSED_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2011_03009_b200 import fus
w = fus.medium_preset("water")
out = []
for dims in [(200, 150, 13), (130, 129, 37), (256, 256, 3), (256, 256, 256)]:
    g = fus.make_grid([0, 0, 0], [d * 1e-4 for d in dims], 1e-4, 2)
    k = fus.complex_wavenumber(w, 1.1e6, 2)
    f = fus.random_vector(g.count(), 17)
    out.append(fus.GreenKernel(g, k).apply(f).cpu().numpy())
np.savez(sys.argv[2], *out)
"""


@pytest.mark.parametrize("fused", ["0", "1"])
def test_ab_fused_ring_path_is_bitwise_two_pass(tmp_path, fused):
    # Passes A+B through the L2-resident z-slab ring (FUSG_AB_FUSED=1, opt-in) run the same
    # 16x16x2 tiles as the two separate launches: results must agree bit for bit.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for v in ("0", fused):
        p = tmp_path / f"u{v}.npz"
        env = dict(os.environ, FUSG_AB_FUSED=v)
        r = subprocess.run([sys.executable, "-c", _AB_FUSED_CHILD, root, str(p)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[v] = np.load(p)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res[fused][key])


_QUADTM_CHILD = """
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2011_03009_b200 import fus
w = fus.medium_preset("water")
out = []
# Pz = 1536 with full and partial rows, odd / even / tiny Px, Py (self-mirror lines, idle warps)
for dims in [(5, 4, 768), (1, 1, 700), (12, 9, 650), (33, 2, 601), (40, 37, 768)]:
    g = fus.make_grid([0, 0, 0], [d * 1e-4 for d in dims], 1e-4, 2)
    assert fus.padded_dims(g)[2] == 1536
    k = fus.complex_wavenumber(w, 1.1e6, 2)
    f = fus.random_vector(g.count(), 23)
    K = fus.GreenKernel(g, k)
    out.append(K.apply(f, -0.5).cpu().numpy())
    out.append(K.apply(f).cpu().numpy())
np.savez(sys.argv[2], *out)
"""


@pytest.mark.gpu
def test_quad_cta_tensor_memory_pass_c_is_bitwise_three_warp_kernel(tmp_path):
    # FUSG_X3_QUADTM=1 (opt-in): pass C at 1536 with one 12-warp CTA per folded K^ row and the
    # recombination of the three residues through tensor memory (tcgen05.st / tcgen05.ld) runs
    # the same transforms and the same recombination expressions: bit for bit the default.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for v in ("0", "1"):
        p = tmp_path / f"u{v}.npz"
        env = dict(os.environ, FUSG_X3_QUADTM=v)
        r = subprocess.run([sys.executable, "-c", _QUADTM_CHILD, root, str(p)], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res[v] = np.load(p)
    for key in res["0"].files:
        assert np.array_equal(res["0"][key], res["1"][key]), key


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_incident_field_zslabs_are_bitwise_the_full_field(ctx, G):
    # p1 shards by z-planes with no collective; ragged slabs of any split must
    # reproduce the single-GPU field bit for bit (attenuating water: tabulated attenuation)
    t = fus.transducer_preset("H131", 100.0, 4096)
    w = water()
    plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 2, 0.3)
    g = plan.for_harmonic(2).grid
    full = fus.evaluate_first_harmonic(t, w, g, 3.0).values
    nz = g.dims[2]
    parts, z0 = [], 0
    for r in range(G):
        n = nz // G + (1 if r < nz % G else 0)
        parts.append(fus.evaluate_first_harmonic_zslab(t, w, g, 3.0, z0, n))
        z0 += n
    assert torch.equal(torch.cat(parts), full)
    with pytest.raises(ValueError):
        fus.evaluate_first_harmonic_zslab(t, w, g, 3.0, nz - 1, 2)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_interpolate_zslabs_with_halo_are_bitwise_the_full_transfer(ctx, G):
    # each target z-slab reads one contiguous source plane range (its planes plus
    # a one-plane halo); the slab transfer must reproduce the full transfer bit for bit
    t = fus.transducer_preset("H131", 100.0, 512)
    w = water()
    plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 3, 0.3)
    gs, gt = plan.for_harmonic(2).grid, plan.for_harmonic(3).grid
    f = torch.from_numpy(fus.random_vector(gs.count(), 21)).cuda()
    full = fus.interpolate(fus.HarmonicField(gs, f, fus.complex_wavenumber(w, t.f0, 2)), gt).values
    nxy = gs.dims[0] * gs.dims[1]
    nz = gt.dims[2]
    parts, z0 = [], 0
    for r in range(G):
        n = nz // G + (1 if r < nz % G else 0)
        lo, hi = fus.interpolate_source_planes(gs, gt, z0, n)
        assert 0 <= lo <= hi < gs.dims[2]
        parts.append(fus.interpolate_zslab(gs, f[lo * nxy:(hi + 1) * nxy], lo, gt, z0, n))
        if lo > 0 and n > 0:  # a slab without its first needed plane is refused
            with pytest.raises(ValueError, match="lacks planes"):
                fus.interpolate_zslab(gs, f[(lo + 1) * nxy:(hi + 1) * nxy], lo + 1, gt, z0, n)
        z0 += n
    assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("G,transport", [(1, "auto"), (2, "auto"), (3, "nccl"), (4, "auto")])
def test_cascade_zslab_loopback_is_bitwise_run_cascade(ctx, G, transport):
    # the cascade decomposed into z-slabs (incident field per slab, halo
    # transfers, slab-sharded applies) reproduces the single-GPU cascade bit for bit
    t = fus.transducer_preset("H131", 100.0, 512)
    w = water()
    plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 3, 0.3)
    cfg = fus.CascadeConfig(w, t, plan, 3)
    want = fus.run_cascade(cfg)
    got = fus.run_cascade_zslab_loopback(cfg, G, transport=transport)
    assert got.source_normalization == want.source_normalization
    for a, b in zip(got.harmonics, want.harmonics):
        assert torch.equal(a.values, b.values)


def test_apply_scale_and_host_path_on_the_512_kernels(ctx):
    # The 16x16x2 kernels at padded length 512 on every axis: the scale argument is applied at
    # the final store (a power of two scales exactly), and the z-chunked host-vector apply runs
    # the same kernels (bitwise equal to the device apply).
    dx = 1e-4
    dims = (254, 253, 230)  # 2N - 1 > 504: every axis pads to 512
    g = fus.make_grid([0, 0, 0], [d * dx for d in dims], dx, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    K = fus.GreenKernel(g, k)
    assert K.padded == (512, 512, 512)
    f = fus.random_vector(g.count(), 33)
    u = K.apply(f)
    assert torch.equal(K.apply(f, -0.5), -0.5 * u)
    assert np.array_equal(K.apply_host(f), host(u))


_ATT_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2011_03009_b200 import fus
t = fus.transducer_preset("H131", 100.0, 1024)
w = fus.medium_preset("water")
plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 2, 0.3)
g = plan.for_harmonic(2).grid
np.save(sys.argv[2], fus.evaluate_first_harmonic(t, w, g, 3.0).values.cpu().numpy())
"""


def test_tabulated_attenuation_matches_the_polynomial_and_exp_paths(tmp_path):
    # The Rayleigh grid kernel's tabulated e^{-Im k d} (FUSG_ATT_TABLE=1, default) against the
    # degree-6 interpolant / exp() modes (FUSG_ATT_TABLE=0) on an attenuating medium
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("1", "0"):
        p = tmp_path / f"p{v}.npy"
        r = subprocess.run([sys.executable, "-c", _ATT_CHILD, root, str(p)], env=dict(os.environ, FUSG_ATT_TABLE=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = np.load(p)
    assert rel_l2(out["1"], out["0"]) <= 1e-13


@pytest.mark.parametrize("transport", ["nccl", "auto"])
def test_multiprocess_zslab_cascade_single_rank_is_bitwise_run_cascade(transport):
    # The multi-process sharded cascade (paper_2011_03009_b200/zslab.py) on a one-rank NCCL
    # communicator: every piece runs (slab incident field, halo plan, slab transfers, rhs, the
    # slab-sharded apply with its NCCL / IPC machinery); bitwise = run_cascade.
    from paper_2011_03009_b200 import zslab

    med, t, k1 = _reduced_cfg4(fus)
    t.power = fus.radiated_power(t, med, k1, 2.0 * k1.k.real * 1.0e6)
    cfg = fus.CascadeConfig(med, t, fus.plan_nested_meshes(t, med, 10.2e-3, 6, 4), 4)
    want = fus.run_cascade(cfg)
    c = fus.Context(0)
    fus.attach_nccl(c, 1, 0, fus.nccl_unique_id())
    got = zslab.run_cascade_zslab(cfg, zslab.Comm(), c, transport)
    assert got.source_normalization == want.source_normalization
    for n in range(1, 5):
        assert got.slabs_z[n - 1] == (0, want.p(n).grid.dims[2])
        assert torch.equal(got.slabs[n - 1], want.p(n).values), n
    assert [row["harmonic"] for row in got.rows] == [2, 3, 4]


def test_context_outlives_its_kernels_in_any_release_order():
    # Owners may be released in any order (e.g. Python finalising a traceback's frames): the
    # context is freed with its last kernel, not under a live one.
    from paper_2011_03009_b200 import _lib

    L = _lib.lib()
    c = fus.Context(0)
    g = fus.make_grid([0, 0, 0], [16e-4, 12e-4, 8e-4], 1e-4, 2)
    k = fus.complex_wavenumber(water(), 1.1e6, 2)
    K = fus.GreenKernel(g, k, ctx=c)
    f = fus.random_vector(g.count(), 3)
    want = K.apply(f).clone()
    L.fusg_ctx_destroy(c.handle)  # the owner lets go first
    c.handle = None
    fd = torch.from_numpy(f).cuda()
    u = torch.empty_like(fd)
    _lib.check(L.fusg_kernel_apply(K.handle, fd.data_ptr(), u.data_ptr(), 1.0, None))  # still works
    torch.cuda.synchronize()
    assert torch.equal(u, want)
    del K  # and frees the context with it
