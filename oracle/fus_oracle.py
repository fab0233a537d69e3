"""ORACLE — TEST INFRASTRUCTURE ONLY (never the product path).

CPU restatement of the fus-harmonics reference (arXiv 2011.03009, C++ tree at
/root/reference/proj) for the volume-potential hot path.  Loops live in ``fus_oracle.cpp``
(compiled to ``liboracle.so`` by ``oracle/Makefile``); the 3D DFTs use numpy's pocketfft on
exactly the reference's padded box, standing in for FFTW (``src/potential.cpp:20-34``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this module.  Pinned against the reference's own known-answer tests and recorded goldens
(``tests/test_oracle_*.py``; list in DESIGN.md §Oracle).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so from fus_oracle.cpp (g++, -ffp-contract=off, OpenMP)."""
    src = os.path.join(_HERE, "fus_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess

        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.orc_last_error.restype = C.c_char_p
        L.orc_random_vector.argtypes = [C.c_int64, C.c_uint, dp]
        L.orc_make_grid.argtypes = [dp, dp, C.c_double, dp, dp, dp, ip]
        L.orc_equivalent_sphere_radius.argtypes = [C.c_double]
        L.orc_equivalent_sphere_radius.restype = C.c_double
        L.orc_self_weight.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.orc_green.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.orc_kernel_fill.argtypes = [ip, ip, C.c_double, C.c_double, C.c_double, dp]
        L.orc_direct_potential.argtypes = [dp, dp, C.c_double, ip, C.c_double, C.c_double, dp, dp]
        L.orc_direct_potential_at.argtypes = [dp, dp, C.c_double, ip, C.c_double, C.c_double, dp,
                                              C.POINTER(C.c_int64), C.c_int64, dp]
        L.orc_evaluate_potential_at.argtypes = [C.c_double, C.c_double, dp, dp, C.c_double, ip, dp,
                                                dp, C.c_int64, dp]
        L.orc_distribute_points.argtypes = [C.c_double, C.c_double, C.c_int, dp]
        L.orc_monopole_points.argtypes = [dp, C.c_int, dp, C.c_int64, C.c_double, C.c_double,
                                          C.c_double, dp]
        L.orc_monopole_grid.argtypes = [dp, C.c_int, dp, dp, C.c_double, ip, C.c_double,
                                        C.c_double, C.c_double, dp]
        L.orc_radiated_power.argtypes = [dp, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                         C.c_int, dp]
        L.orc_interpolate.argtypes = [dp, dp, C.c_double, ip, dp, dp, dp, C.c_double, ip, dp]
        L.orc_rhs_source.argtypes = [C.c_int, C.POINTER(dp), C.c_int64, C.c_double, C.c_double,
                                     C.c_double, C.c_double, dp]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32).ctypes.data_as(C.POINTER(C.c_int))


def _check(rc: int, exc=ValueError):
    if rc:
        raise exc(lib().orc_last_error().decode())


# --------------------------------------------------------------------------- L1 types
@dataclass
class Medium:
    """include/fus/medium.hpp:12-23"""
    name: str
    rho0: float
    c0: float
    beta: float
    alpha0: float
    eta: float


@dataclass
class Wavenumber:
    """include/fus/medium.hpp:26-30"""
    k: complex
    harmonic: int
    omega: float


K_DB_PER_NEPER = 8.685889638065035  # include/fus/medium.hpp:33


def medium_preset(name: str) -> Medium:
    """src/medium.cpp:47-52"""
    if name == "water":
        return Medium("water", 1000.0, 1480.0, 3.5, 0.2, 2.0)
    if name == "liver":
        return Medium("liver", 1060.0, 1590.0, 4.4, 90.0, 1.1)
    if name == "kidney":
        return Medium("kidney", 1050.0, 1570.0, 4.7, 10.0, 1.0)
    raise ValueError(f"unknown medium preset '{name}'")


def attenuation_np_per_m(m: Medium, f_hz: float) -> float:
    """src/medium.cpp:25-29"""
    f_mhz = f_hz / 1.0e6
    return m.alpha0 * math.pow(f_mhz, m.eta) / K_DB_PER_NEPER


def complex_wavenumber(m: Medium, f0: float, n: int) -> Wavenumber:
    """src/medium.cpp:31-45"""
    if f0 <= 0.0:
        raise ValueError("complex_wavenumber: f0 must be positive")
    if n < 1:
        raise ValueError("complex_wavenumber: harmonic index must be >= 1")
    omega = 2.0 * math.pi * f0
    alpha = attenuation_np_per_m(m, n * f0)
    return Wavenumber(complex(n * omega / m.c0, alpha), n, omega)


@dataclass
class VoxelGrid:
    """include/fus/grid.hpp:30-50 (x fastest)."""
    lo: np.ndarray
    hi: np.ndarray
    dx: float
    dims: tuple
    harmonic: int = 1

    def count(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def index(self, ix, iy, iz) -> int:
        return ix + self.dims[0] * (iy + self.dims[1] * iz)

    def center(self, ix, iy, iz) -> np.ndarray:
        return np.array([self.lo[0] + (ix + 0.5) * self.dx, self.lo[1] + (iy + 0.5) * self.dx,
                         self.lo[2] + (iz + 0.5) * self.dx])

    def centers_axis(self, a: int) -> np.ndarray:
        return self.lo[a] + (np.arange(self.dims[a]) + 0.5) * self.dx

    def args(self):
        return _d(self.lo), _d(self.hi), float(self.dx), _i(self.dims)


def make_grid(lo, hi, dx: float, harmonic: int, anchor=None) -> VoxelGrid:
    """src/grid.cpp:12-34"""
    olo, ohi, odims = np.zeros(3), np.zeros(3), np.zeros(3, np.int32)
    anc = _d(np.asarray(anchor, float)) if anchor is not None else None
    rc = lib().orc_make_grid(_d(lo), _d(hi), float(dx), anc, olo.ctypes.data_as(C.POINTER(C.c_double)),
                             ohi.ctypes.data_as(C.POINTER(C.c_double)),
                             odims.ctypes.data_as(C.POINTER(C.c_int)))
    _check(rc)
    return VoxelGrid(olo, ohi, float(dx), tuple(int(v) for v in odims), harmonic)


@dataclass
class HarmonicField:
    """include/fus/grid.hpp:57-61"""
    grid: VoxelGrid
    values: np.ndarray  # complex128, size grid.count(), x fastest
    wavenumber: Wavenumber


def random_vector(n: int, seed: int) -> np.ndarray:
    """tests/acceptance.cpp:30-36 (libstdc++ mt19937 + uniform_real_distribution)."""
    out = np.empty(2 * n, np.float64)
    lib().orc_random_vector(n, seed, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out.view(np.complex128)


# --------------------------------------------------------------------------- potential
def equivalent_sphere_radius(dx: float) -> float:
    return lib().orc_equivalent_sphere_radius(dx)


def self_weight(k: Wavenumber, dx: float) -> complex:
    """src/potential.cpp:59-70"""
    out = np.zeros(2)
    _check(lib().orc_self_weight(k.k.real, k.k.imag, dx, _dp(out)))
    return complex(out[0], out[1])


def green_function(x, y, k: Wavenumber) -> complex:
    """src/potential.cpp:47-53"""
    d = np.asarray(x, float) - np.asarray(y, float)
    r = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    if r < 1e-300:
        raise ValueError("green_function: singular at x == y")
    out = np.zeros(2)
    lib().orc_green(k.k.real, k.k.imag, r, _dp(out))
    return complex(out[0], out[1])


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def next_fast_size(n: int) -> int:
    """src/potential.cpp:36-43"""
    while True:
        m = n
        for p in (2, 3, 5, 7):
            while m % p == 0:
                m //= p
        if m == 1:
            return n
        n += 1


class GreenKernel:
    """src/potential.cpp:72-159.  ``padded`` defaults to the reference's choice (2N, or
    next_fast_size(2N)); any P >= 2N-1 is mathematically identical (offset_of, :88-94), which
    lets the parity tests run the oracle on the GPU path's own padded box too."""

    def __init__(self, grid: VoxelGrid, k: Wavenumber, pad_small_primes: bool = False,
                 padded: Optional[Sequence[int]] = None, workers: int = 1):
        self.grid, self.k, self.workers = grid, k, workers
        if padded is None:
            padded = [next_fast_size(2 * n) if pad_small_primes else 2 * n for n in grid.dims]
        self.padded = tuple(int(p) for p in padded)
        P = self.padded
        buf = np.empty(2 * P[0] * P[1] * P[2], np.float64)
        _check(lib().orc_kernel_fill(_i(grid.dims), _i(P), grid.dx, k.k.real, k.k.imag, _dp(buf)))
        kt = buf.view(np.complex128).reshape(P[2], P[1], P[0])
        self.kernel_hat = _fftn(kt, workers)

    def apply(self, f: np.ndarray) -> np.ndarray:
        n = self.grid.dims
        if f.size != self.grid.count():
            raise ValueError("GreenKernel::apply: field size does not match kernel grid")
        P = self.padded
        work = np.zeros((P[2], P[1], P[0]), np.complex128)
        work[: n[2], : n[1], : n[0]] = np.asarray(f).reshape(n[2], n[1], n[0])
        work = _fftn(work, self.workers)
        work *= self.kernel_hat
        work = _ifftn_unnormalised(work, self.workers)
        work /= float(P[0] * P[1] * P[2])
        return np.ascontiguousarray(work[: n[2], : n[1], : n[0]]).reshape(-1)

    def apply_field(self, f: HarmonicField) -> HarmonicField:
        return HarmonicField(self.grid, self.apply(f.values), self.k)


class SampledApply:
    """Bounded sample of GreenKernel::apply (src/potential.cpp:128-149) for boxes too large to
    run whole within a benchmark's time budget ("time a stated fraction
    and report it as extrapolated").  The reference's apply is pad -> 3D FFT of the P box ->
    multiply by the P-box spectrum -> inverse 3D FFT -> /|P| -> crop; its 3D FFTs are three
    batches of one-dimensional transforms (one batch per axis).  One sample runs `planes`
    z-planes' share of every stage at the full line lengths and strides:
      * pad + crop + the spectrum multiply + the 1/|P| scale on a (planes, Py, Px) block;
      * forward and inverse x-line and y-line transforms on that block;
      * forward and inverse z-line transforms on a (Pz, planes*Py/Pz, Px) block.
    That is the fraction F = planes/Pz of every stage's lines, so t_apply = t_sample / F.
    Inputs are the first `planes` z-planes of the seeded source (random_vector(n, seed) is
    sequential in x-fastest order); the multiply's factor block holds stand-in values (the
    timing does not depend on them)."""

    def __init__(self, dims, P, planes: int, workers: int, seed: int):
        self.n = [int(v) for v in dims]
        self.P = [int(v) for v in P]
        self.planes = max(1, min(int(planes), self.P[2]))
        self.workers = workers
        n, P = self.n, self.P
        self.nzf = min(self.planes, n[2])
        self.f = random_vector(self.nzf * n[1] * n[0], seed).reshape(self.nzf, n[1], n[0])
        self.khat = np.full((self.planes, P[1], P[0]), 1.0 + 0.5j, np.complex128)
        self.zcols = max(1, self.planes * P[1] // P[2])
        self.zb = np.ones((P[2], self.zcols, P[0]), np.complex128)
        self.fraction = self.planes / P[2]

    def run(self) -> float:
        """One sample; returns its seconds."""
        import scipy.fft as sf

        n, P, w = self.n, self.P, self.workers
        t0 = __import__("time").perf_counter()
        work = np.zeros((self.planes, P[1], P[0]), np.complex128)  # pad (:130-134)
        work[: self.nzf, : n[1], : n[0]] = self.f
        for ax in (2, 1):  # forward x, y lines of the block
            work = sf.fft(work, axis=ax, workers=w, overwrite_x=True)
        self.zb = sf.fft(self.zb, axis=0, workers=w, overwrite_x=True)  # forward z lines
        work *= self.khat  # (:137-139)
        self.zb = sf.ifft(self.zb, axis=0, norm="forward", workers=w, overwrite_x=True)
        for ax in (1, 2):
            work = sf.ifft(work, axis=ax, norm="forward", workers=w, overwrite_x=True)
        work /= float(P[0] * P[1] * P[2])  # (:141)
        out = np.ascontiguousarray(work[: self.nzf, : n[1], : n[0]])  # crop (:143-149)
        dt = __import__("time").perf_counter() - t0
        del out, work
        return dt


def sampled_apply_seconds(dims, P, planes: int, workers: int, seed: int, reps: int = 1):
    """(seconds per extrapolated apply, fraction, best seconds per sample) of SampledApply."""
    s = SampledApply(dims, P, planes, workers, seed)
    best = min(s.run() for _ in range(max(1, reps)))
    return best / s.fraction, s.fraction, best


def _fftn(a, workers):
    try:
        import scipy.fft as sf

        return sf.fftn(a, workers=workers)
    except ImportError:  # pragma: no cover
        return np.fft.fftn(a)


def _ifftn_unnormalised(a, workers):
    try:
        import scipy.fft as sf

        return sf.ifftn(a, norm="forward", workers=workers)
    except ImportError:  # pragma: no cover
        return np.fft.ifftn(a, norm="forward")


def direct_potential_oracle(k: Wavenumber, grid: VoxelGrid, f: np.ndarray) -> np.ndarray:
    """src/potential.cpp:203-238"""
    if f.size != grid.count():
        raise ValueError("direct_potential_oracle: field size mismatch")
    out = np.empty(grid.count(), np.complex128)
    f = np.ascontiguousarray(f, np.complex128)
    lo, hi, dx, dims = grid.args()
    _check(lib().orc_direct_potential(lo, hi, dx, dims, k.k.real, k.k.imag,
                                      _dp(f.view(np.float64)), _dp(out.view(np.float64))))
    return out


def direct_potential_at(k: Wavenumber, grid: VoxelGrid, f: np.ndarray, indices) -> np.ndarray:
    """direct_potential_oracle (src/potential.cpp:203-238) at the voxels `indices` only (O(N)
    per output): checks full-size applies at sampled voxels."""
    if f.size != grid.count():
        raise ValueError("direct_potential_at: field size mismatch")
    f = np.ascontiguousarray(f, np.complex128)
    idx = np.ascontiguousarray(indices, np.int64)
    out = np.empty(idx.size, np.complex128)
    lo, hi, dx, dims = grid.args()
    _check(lib().orc_direct_potential_at(lo, hi, dx, dims, k.k.real, k.k.imag, _dp(f.view(np.float64)),
                                         idx.ctypes.data_as(C.POINTER(C.c_int64)), idx.size,
                                         _dp(out.view(np.float64))))
    return out


def evaluate_potential_at(k: Wavenumber, grid: VoxelGrid, f: np.ndarray, points) -> np.ndarray:
    """src/potential.cpp:161-201"""
    if f.size != grid.count():
        raise ValueError("evaluate_potential_at: field size mismatch")
    pts = np.ascontiguousarray(np.asarray(points, float).reshape(-1, 3))
    out = np.empty(len(pts), np.complex128)
    f = np.ascontiguousarray(f, np.complex128)
    lo, hi, dx, dims = grid.args()
    _check(lib().orc_evaluate_potential_at(k.k.real, k.k.imag, lo, hi, dx, dims,
                                           _dp(f.view(np.float64)), _dp(pts), len(pts),
                                           _dp(out.view(np.float64))))
    return out


# --------------------------------------------------------------------------- transducer
@dataclass
class BowlTransducer:
    """include/fus/transducer.hpp:15-28"""
    name: str
    f0: float
    focal_length: float
    outer_radius: float
    power: float
    source_points: np.ndarray  # (n_p, 3)

    def focus(self):
        return np.array([self.focal_length, 0.0, 0.0])

    def cap_area(self) -> float:
        l, R = self.focal_length, self.outer_radius
        return 2.0 * math.pi * l * (l - math.sqrt(l * l - R * R))

    def rim_plane_x(self) -> float:
        l, R = self.focal_length, self.outer_radius
        return l - math.sqrt(l * l - R * R)


def distribute_points(l: float, R: float, n: int) -> np.ndarray:
    """src/transducer.cpp:22-70"""
    out = np.empty(3 * n, np.float64)
    _check(lib().orc_distribute_points(l, R, n, _dp(out)))
    return out.reshape(n, 3)


def make_bowl(name, f0, l, R, power, n_points) -> BowlTransducer:
    """src/transducer.cpp:72-84"""
    if f0 <= 0.0:
        raise ValueError("make_bowl: f0 must be positive")
    if power < 0.0:
        raise ValueError("make_bowl: power must be >= 0")
    return BowlTransducer(name, f0, l, R, power, distribute_points(l, R, n_points))


def transducer_preset(name: str, power: float = 100.0, n_points: int = 4096) -> BowlTransducer:
    """src/transducer.cpp:86-92"""
    if name == "H101":
        return make_bowl("H101", 1.1e6, 63.2e-3, 32.0e-3, power, n_points)
    if name == "H131":
        return make_bowl("H131", 1.1e6, 35.0e-3, 16.5e-3, power, n_points)
    raise ValueError(f"unknown transducer preset '{name}'")


def unnormalized_field(t: BowlTransducer, pts, k: Wavenumber, amp: Optional[float] = None):
    """src/transducer.cpp:123-132"""
    if amp is None:
        amp = t.cap_area() / float(len(t.source_points))
    pts = np.ascontiguousarray(np.asarray(pts, float).reshape(-1, 3))
    out = np.empty(len(pts), np.complex128)
    src = np.ascontiguousarray(t.source_points, np.float64)
    _check(lib().orc_monopole_points(_dp(src), len(src), _dp(pts), len(pts), k.k.real, k.k.imag,
                                     amp, _dp(out.view(np.float64))))
    return out


def radiated_power(t: BowlTransducer, m: Medium, k: Wavenumber, amplitude_scale: float,
                   n_r: int = 384, n_theta: int = 256) -> float:
    """src/transducer.cpp:134-155"""
    amp = amplitude_scale * t.cap_area() / float(len(t.source_points))
    src = np.ascontiguousarray(t.source_points, np.float64)
    out = np.zeros(1)
    _check(lib().orc_radiated_power(_dp(src), len(src), t.rim_plane_x(), t.outer_radius,
                                    k.k.real, k.k.imag, amp, m.rho0, m.c0, n_r, n_theta,
                                    _dp(out)))
    return float(out[0])


def power_scale_factor(t: BowlTransducer, m: Medium, k: Wavenumber) -> float:
    """src/transducer.cpp:157-163"""
    if t.power == 0.0:
        return 0.0
    pw = radiated_power(t, m, k, 1.0)
    if pw <= 0.0:
        raise RuntimeError("power normalization: degenerate field, Pi(p) = 0")
    return math.sqrt(t.power / pw)


def evaluate_first_harmonic(t: BowlTransducer, m: Medium, grid: VoxelGrid,
                            amplitude_scale: float) -> HarmonicField:
    """src/transducer.cpp:179-196"""
    k1 = complex_wavenumber(m, t.f0, 1)
    amp = amplitude_scale * t.cap_area() / float(len(t.source_points))
    src = np.ascontiguousarray(t.source_points, np.float64)
    out = np.empty(grid.count(), np.complex128)
    lo, hi, dx, dims = grid.args()
    _check(lib().orc_monopole_grid(_dp(src), len(src), lo, hi, dx, dims, k1.k.real, k1.k.imag,
                                   amp, _dp(out.view(np.float64))))
    return HarmonicField(grid, out, k1)


def evaluate_source_field(t: BowlTransducer, m: Medium, grid: VoxelGrid):
    """src/transducer.cpp:198-206 -> (field, normalization)"""
    k1 = complex_wavenumber(m, t.f0, 1)
    scale = power_scale_factor(t, m, k1)
    f = evaluate_first_harmonic(t, m, grid, scale)
    return f, (scale if scale > 0.0 else 1.0)


# --------------------------------------------------------------------------- planner
@dataclass
class PlannedGrid:
    harmonic: int
    domain_lo: np.ndarray
    domain_hi: np.ndarray
    grid: VoxelGrid


@dataclass
class MeshPlan:
    """include/fus/grid.hpp:71-84"""
    grids: List[PlannedGrid]
    reference: VoxelGrid
    d: float
    w: float
    focus: np.ndarray
    n_w: int

    def for_harmonic(self, n: int) -> PlannedGrid:
        for pg in self.grids:
            if pg.harmonic == n:
                return pg
        raise IndexError(f"MeshPlan: no grid planned for harmonic {n}")

    def reduction_factor(self, n: int) -> float:
        return float(self.reference.count()) / float(self.for_harmonic(n).grid.count())


def reference_domain(t: BowlTransducer, d: float):
    """src/grid.cpp:70-79"""
    if d < 0.0:
        raise ValueError("reference_domain: d must be >= 0")
    l, R = t.focal_length, t.outer_radius
    L = math.sqrt(l * l - R * R) - 0.1e-3
    return np.array([l - L, -R, -R]), np.array([l + d, R, R])


def plan_nested_meshes(t: BowlTransducer, m: Medium, d: float, n_w: int, n_harmonics: int,
                       width_scale: float = 1.0) -> MeshPlan:
    """src/grid.cpp:81-112"""
    if n_harmonics < 2:
        raise ValueError("plan_nested_meshes: need n_harmonics >= 2")
    if n_w < 1:
        raise ValueError("plan_nested_meshes: need n_w >= 1")
    lambda1 = m.c0 / t.f0
    focus = t.focus()
    ref_lo, _ = reference_domain(t, d)
    L = focus[0] - ref_lo[0]
    w = 2.0 * t.outer_radius * width_scale
    d2_lo = np.array([focus[0] - L, -w / 2.0, -w / 2.0])
    d2_hi = np.array([focus[0] + d, w / 2.0, w / 2.0])
    reference = make_grid(d2_lo, d2_hi, lambda1 / (n_harmonics * n_w), n_harmonics, focus)
    grids = []
    for i in range(2, n_harmonics + 1):
        s = 2.0 / float(i)
        lo = np.array([focus[0] - s * L, -s * w / 2.0, -s * w / 2.0])
        hi = np.array([focus[0] + d, s * w / 2.0, s * w / 2.0])
        grids.append(PlannedGrid(i, lo, hi, make_grid(lo, hi, lambda1 / (i * n_w), i, focus)))
    return MeshPlan(grids, reference, d, w, focus, n_w)


def plan_single_mesh(t, m, d, n_w, n_harmonics, width_scale=1.0) -> MeshPlan:
    """src/cascade.cpp:109-118"""
    plan = plan_nested_meshes(t, m, d, n_w, n_harmonics, width_scale)
    first = plan.grids[0]
    for pg in plan.grids:
        pg.domain_lo, pg.domain_hi = first.domain_lo.copy(), first.domain_hi.copy()
        pg.grid = replace(plan.reference, harmonic=pg.harmonic)
    return plan


def interpolate(fld: HarmonicField, target: VoxelGrid) -> HarmonicField:
    """src/grid.cpp:141-195"""
    src = fld.grid
    if fld.values.size != src.count():
        raise ValueError("interpolate: field size does not match its grid")
    out = np.empty(target.count(), np.complex128)
    f = np.ascontiguousarray(fld.values, np.complex128)
    slo, shi, sdx, sdims = src.args()
    tlo, thi, tdx, tdims = target.args()
    _check(lib().orc_interpolate(slo, shi, sdx, sdims, _dp(f.view(np.float64)), tlo, thi, tdx,
                                 tdims, _dp(out.view(np.float64))))
    return HarmonicField(target, out, fld.wavenumber)


# --------------------------------------------------------------------------- cascade
def rhs_source(n: int, lower: List[HarmonicField], m: Medium, omega: float) -> np.ndarray:
    """src/cascade.cpp:21-40"""
    if n < 2:
        raise ValueError("rhs_source: harmonic index must be >= 2")
    if len(lower) < n - 1:
        raise ValueError(f"rhs_source: missing lower harmonics for n = {n}")
    count = lower[0].values.size
    for i in range(n - 1):
        if lower[i].values.size != count:
            raise ValueError("rhs_source: lower harmonics live on different grids")
    arrs = [np.ascontiguousarray(h.values, np.complex128) for h in lower[: n - 1]]
    ptrs = (C.POINTER(C.c_double) * len(arrs))(*[_dp(a.view(np.float64)) for a in arrs])
    out = np.empty(count, np.complex128)
    lib().orc_rhs_source(n, ptrs, count, m.beta, omega, m.rho0, m.c0, _dp(out.view(np.float64)))
    return out


def rhs_source_full(n: int, fields: List[HarmonicField], m: Medium, omega: float) -> np.ndarray:
    """The paper's full quadratic source, Eq. (cascade_1), truncated at
    M = len(fields) harmonics: coeff * [sum_{m=1}^{n-1} p_m p_{n-m} + 2 sum_{m=n+1}^{M} p_m conj(p_{m-n})].
    The reference implements only the first sum (src/cascade.cpp:36-39), so this is parity
    unpinned beyond M = n - 1; plain numpy in the device kernel's accumulation order."""
    M = len(fields)
    coeff = m.beta * omega * omega * n * n / (2.0 * m.rho0 * m.c0 ** 4)  # src/cascade.cpp:32-34
    count = fields[0].values.size
    re = np.zeros(count)
    im = np.zeros(count)
    for k in range(1, n):
        a, b = fields[k - 1].values, fields[n - k - 1].values
        re = re + (a.real * b.real - a.imag * b.imag)
        im = im + (a.real * b.imag + a.imag * b.real)
    for k in range(n + 1, M + 1):
        a, b = fields[k - 1].values, fields[k - n - 1].values
        re = re + 2.0 * (a.real * b.real + a.imag * b.imag)
        im = im + 2.0 * (a.imag * b.real - a.real * b.imag)
    return coeff * re + 1j * (coeff * im)


def same_grid(a: VoxelGrid, b: VoxelGrid) -> bool:
    """src/cascade.cpp:15-17"""
    return tuple(a.dims) == tuple(b.dims) and a.dx == b.dx and bool(np.all(a.lo == b.lo))


@dataclass
class CascadeConfig:
    """include/fus/cascade.hpp:12-21"""
    medium: Medium
    transducer: BowlTransducer
    plan: MeshPlan
    n_harmonics: int = 5
    recompute_p1_each_grid: bool = False
    pad_small_primes: bool = False


@dataclass
class CascadeResult:
    harmonics: List[HarmonicField] = field(default_factory=list)
    source_normalization: float = 1.0

    def p(self, n: int) -> HarmonicField:
        return self.harmonics[n - 1]


def run_cascade(cfg: CascadeConfig, padded_for=None, workers: int = 1) -> CascadeResult:
    """src/cascade.cpp:42-107.  ``padded_for(grid)`` optionally picks the padded box (any
    P >= 2N-1 is exact); default is the reference's own choice."""
    plan, n = cfg.plan, cfg.n_harmonics
    if n < 2:
        raise ValueError("run_cascade: n_harmonics must be >= 2")
    res = CascadeResult()
    p1, norm = evaluate_source_field(cfg.transducer, cfg.medium, plan.for_harmonic(2).grid)
    res.source_normalization = norm
    res.harmonics.append(p1)
    for i in range(2, n + 1):
        grid = plan.for_harmonic(i).grid
        lower = []
        for mm in range(1, i):
            pm = res.harmonics[mm - 1]
            if same_grid(pm.grid, grid):
                lower.append(pm)
            elif mm == 1 and cfg.recompute_p1_each_grid:
                lower.append(evaluate_first_harmonic(cfg.transducer, cfg.medium, grid,
                                                     res.source_normalization))
            else:
                lower.append(interpolate(pm, grid))
        ki = complex_wavenumber(cfg.medium, cfg.transducer.f0, i)
        f = rhs_source(i, lower, cfg.medium, ki.omega)
        padded = padded_for(grid) if padded_for else None
        kern = GreenKernel(grid, ki, cfg.pad_small_primes, padded=padded, workers=workers)
        res.harmonics.append(HarmonicField(grid, -kern.apply(f), ki))
    return res


# --------------------------------------------------------------------------- analysis helpers
def extract_on_axis(fld: HarmonicField):
    """src/analysis.cpp:49-68 -> (x, p)"""
    g = fld.grid

    def axis_weights(lo, dx, n):
        q = (0.0 - lo) / dx - 0.5
        j0 = int(math.floor(q))
        if j0 < 0:
            j0 = 0
        if j0 > n - 2:
            j0 = max(0, n - 2)
        t = q - j0
        if t < 0.0:
            t = 0.0
        if t > 1.0:
            t = 1.0 if n > 1 else 0.0
        return j0, t

    jy, ty = axis_weights(g.lo[1], g.dx, g.dims[1])
    jz, tz = axis_weights(g.lo[2], g.dx, g.dims[2])
    jy1, jz1 = min(jy + 1, g.dims[1] - 1), min(jz + 1, g.dims[2] - 1)
    v = fld.values.reshape(g.dims[2], g.dims[1], g.dims[0])
    x = g.lo[0] + (np.arange(g.dims[0]) + 0.5) * g.dx
    p = ((1.0 - ty) * (1.0 - tz) * v[jz, jy, :] + ty * (1.0 - tz) * v[jz, jy1, :] +
         (1.0 - ty) * tz * v[jz1, jy, :] + ty * tz * v[jz1, jy1, :])
    return x, p


def _resample(px, pp, nodes):
    """src/analysis.cpp:27-45"""
    out = np.empty(len(nodes), np.complex128)
    for i, x in enumerate(nodes):
        if x <= px[0]:
            out[i] = pp[0]
        elif x >= px[-1]:
            out[i] = pp[-1]
        else:
            j = int((x - px[0]) / (px[1] - px[0]))
            while j + 1 < len(px) and px[j + 1] < x:
                j += 1
            while j > 0 and px[j] > x:
                j -= 1
            t = (x - px[j]) / (px[j + 1] - px[j])
            out[i] = (1.0 - t) * pp[j] + t * pp[j + 1]
    return out


def on_axis_error(p, p_ref, normalizer) -> float:
    """src/analysis.cpp:70-78; profiles are (x, p) tuples."""
    a = _resample(p[0], p[1], p_ref[0])
    nrm = _resample(normalizer[0], normalizer[1], p_ref[0])
    denom = float(np.linalg.norm(nrm))
    if denom == 0.0:
        raise ValueError("on_axis_error: normalizer has zero norm")
    return 100.0 * float(np.linalg.norm(a - p_ref[1])) / denom


def quadrature_convergence_study(t, m, box_lo, box_hi, n_w_values, n_w_ref):
    """src/analysis.cpp:92-162 -> (records [(n_w, err%)], slope)"""
    for nw in n_w_values:
        if nw >= n_w_ref:
            raise ValueError("quadrature_convergence_study: n_w_ref must exceed all n_w")
    lambda1 = m.c0 / t.f0
    k1 = complex_wavenumber(m, t.f0, 1)
    k2 = complex_wavenumber(m, t.f0, 2)
    scale = power_scale_factor(t, m, k1)

    def source(nw):
        grid = make_grid(box_lo, box_hi, lambda1 / (2.0 * nw), 2)
        lower = [evaluate_first_harmonic(t, m, grid, scale)]
        return grid, rhs_source(2, lower, m, k2.omega)

    g, f = source(n_w_ref)
    ref_x = g.lo[0] + (np.arange(g.dims[0]) + 0.5) * g.dx
    nodes = np.stack([ref_x, np.zeros_like(ref_x), np.zeros_like(ref_x)], axis=1)
    ref = (ref_x, -evaluate_potential_at(k2, g, f, nodes))
    records = []
    sx = sy = sxx = sxy = 0.0
    fitted = 0
    for nw in n_w_values:
        g, f = source(nw)
        prof = (ref_x, -evaluate_potential_at(k2, g, f, nodes))
        err = on_axis_error(prof, ref, ref)
        records.append((nw, err))
        if err > 0.0:
            lx, ly = math.log(float(nw)), math.log(err)
            sx += lx
            sy += ly
            sxx += lx * lx
            sxy += lx * ly
            fitted += 1
    slope = (fitted * sxy - sx * sy) / (fitted * sxx - sx * sx) if fitted >= 2 else 0.0
    return records, slope
