"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/fusg.h declares, and its host arithmetic is bit-identical to the pinned oracle."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2011_03009_b200 import _lib, fus

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fusg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"typedef[^;]*;", "", text)  # types (incl. function-pointer typedefs) are not symbols
    return sorted(set(re.findall(r"\b(fusg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding declares exactly the header's entry points
    assert sorted(_lib.SIGNATURES) == syms


def test_no_gpu_needed_for_host_arithmetic():
    assert _lib.lib().fusg_version().startswith(b"fusg")


def test_make_grid_and_plan_bit_exact(orc):
    w, wo = fus.medium_preset("water"), orc.medium_preset("water")
    for name, d, nw, nh, ws in [("H131", 10.2e-3, 6, 5, 1.0), ("H101", 10.2e-3, 6, 5, 1.0),
                                ("H131", 6e-3, 3, 3, 0.35)]:
        t = fus.transducer_preset(name, 100.0, 16)
        to = orc.transducer_preset(name, 100.0, 16)
        for single in (False, True):
            p = (fus.plan_single_mesh if single else fus.plan_nested_meshes)(t, w, d, nw, nh, ws)
            po = (orc.plan_single_mesh if single else orc.plan_nested_meshes)(to, wo, d, nw, nh, ws)
            assert p.reference.dims == po.reference.dims
            assert np.array_equal(p.reference.lo, po.reference.lo)
            for a, b in zip(p.grids, po.grids):
                assert a.grid.dims == b.grid.dims and a.grid.dx == b.grid.dx
                assert np.array_equal(a.grid.lo, b.grid.lo) and np.array_equal(a.grid.hi, b.grid.hi)
                assert np.array_equal(a.domain_lo, b.domain_lo)
    # criterion 5 golden (proj/test_output.txt:31)
    p = fus.plan_nested_meshes(fus.transducer_preset("H131", 100.0, 16), w, 10.2e-3, 6, 5)
    assert p.reference.dims == (914, 737, 737) and p.for_harmonic(2).grid.dims == (366, 295, 295)
    with pytest.raises(IndexError):
        p.for_harmonic(7)
    with pytest.raises(ValueError):
        fus.make_grid([0, 0, 0], [1, 1, 1], -1.0, 1)
    with pytest.raises(ValueError):
        fus.make_grid([0, 0, 0], [1, 0, 1], 0.1, 1)


def test_points_wavenumber_selfweight_bit_exact(orc):
    for n in (1, 7, 128, 4096):
        assert np.array_equal(fus.distribute_points(35e-3, 16.5e-3, n),
                              orc.distribute_points(35e-3, 16.5e-3, n))
    for name in ("water", "liver", "kidney"):
        for n in (1, 2, 5):
            k = fus.complex_wavenumber(fus.medium_preset(name), 1.1e6, n)
            ko = orc.complex_wavenumber(orc.medium_preset(name), 1.1e6, n)
            assert (k.k, k.harmonic, k.omega) == (ko.k, ko.harmonic, ko.omega)
            for dx in (1e-4, 1e-7, 44.85e-6):
                assert fus.self_weight(k, dx) == orc.self_weight(ko, dx)
    with pytest.raises(ValueError):
        fus.complex_wavenumber(fus.medium_preset("water"), -1.0, 1)
    with pytest.raises(ValueError):
        fus.distribute_points(1.0, 2.0, 5)


def test_random_vector_matches_libstdcxx(orc):
    assert np.array_equal(fus.random_vector(1000, 1234), orc.random_vector(1000, 1234))


def test_padded_sizes_are_smooth_and_sufficient():
    for n in list(range(1, 80)) + [256, 487, 518, 768, 1201, 1287, 1333]:
        g = fus.VoxelGrid(np.zeros(3), np.ones(3), 1.0, (n, max(1, n // 2), 1))
        P = fus.padded_dims(g)
        for a in range(3):
            p, N = P[a], g.dims[a]
            assert p >= 2 * N - 1 and p >= 2
            m = p
            for q in (2, 3, 5, 7):
                while m % q == 0:
                    m //= q
            assert m == 1
    assert fus.padded_dims(fus.VoxelGrid(np.zeros(3), np.ones(3), 1.0, (256, 64, 518))) == (512, 128, 1050)


def test_rhs_coefficient_matches_reference_expression():
    w = fus.medium_preset("water")
    om = 2 * math.pi * 1.1e6
    for n in (2, 3, 5):
        want = w.beta * om * om * float(n) * float(n) / (2.0 * w.rho0 * math.pow(w.c0, 4))
        assert _lib.lib().fusg_rhs_coefficient(C.byref(w.c()), om, n) == want


def test_cpp_dropin_api_host_cases():
    """The reference's own host-side cases, compiled against the namespace fus headers
    (include/fus/*.hpp) and linked to libfus.so -> libfusg.so."""
    import subprocess

    exe = os.path.join(ROOT, "build", "test_fus_api")
    assert os.path.exists(exe), "built by __graft_entry__.build() (make -C paper_2011_03009_b200/csrc)"
    out = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK:" in out.stdout


def test_cpp_dropin_test_calls_every_header_declaration():
    """Every function and member function the drop-in headers (include/fus/*.hpp) declare is
    called by the C++ drop-in test (tests/cpp/test_fus_api.cpp), which links only against them."""
    decl = set()
    for name in os.listdir(os.path.join(ROOT, "include", "fus")):
        if name.endswith(".hpp"):
            t = re.sub(r"//.*", "", open(os.path.join(ROOT, "include", "fus", name)).read())
            decl |= {m.group(1) for m in re.finditer(r"^\s*(?:[\w:<>,\s\*&]+?)\s+(\w+)\s*\(", t, re.M)}
    decl -= {"if", "for", "while", "return", "operator"}
    test = open(os.path.join(ROOT, "tests", "cpp", "test_fus_api.cpp")).read()
    missing = sorted(n for n in decl if not re.search(r"\b" + n + r"\b", test))
    assert len(decl) > 60 and not missing, missing


def test_interpolate_source_planes_follow_the_reference_cell_rule():
    # Host restatement (no GPU): the z-slab transfer's source range is the span of the
    # reference's cell bases (src/grid.cpp:156-170: q = (p - lo_s)/dx_s - 0.5,
    # base = clamp(floor q, 0, max(0, n - 2))) and base + 1, over the target slab's planes.
    t = fus.transducer_preset("H131", 100.0, 64)
    w = fus.medium_preset("water")
    plan = fus.plan_nested_meshes(t, w, 6e-3, 2, 4, 0.3)
    for a, b in [(2, 3), (3, 4), (2, 4)]:
        gs, gt = plan.for_harmonic(a).grid, plan.for_harmonic(b).grid
        n = gs.dims[2]
        for z0, nz in [(0, 1), (0, gt.dims[2]), (3, 5), (gt.dims[2] - 2, 2)]:
            bases = []
            for iz in range(z0, z0 + nz):
                p = gt.lo[2] + (iz + 0.5) * gt.dx
                q = (p - gs.lo[2]) / gs.dx - 0.5
                bases.append(min(max(math.floor(q), 0), max(0, n - 2)))
            assert fus.interpolate_source_planes(gs, gt, z0, nz) == (min(bases), min(max(bases) + 1, n - 1))
    with pytest.raises(ValueError):
        fus.interpolate_source_planes(gs, gt, 0, 0)
