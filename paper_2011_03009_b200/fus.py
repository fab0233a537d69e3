"""Python mirror of the reference's ``namespace fus`` API for the volume-potential path.

Same names, argument meaning and error behaviour as ``/root/reference/proj/include/fus/*.hpp``
(ValueError <-> std::invalid_argument, IndexError <-> std::out_of_range, RuntimeError <->
std::runtime_error).  Numerics run in libfusg.so (hand-written sm_100a kernels); host-side
grid/planner arithmetic runs in the same library's bit-exact C++.  Fields are
complex128 torch tensors resident on the GPU; numpy arrays are accepted and copied over.
There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


# ------------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream (fusg_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().fusg_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream_ptr(self) -> int:
        return lib().fusg_ctx_stream(self.handle) or 0

    def synchronize(self):
        check(lib().fusg_ctx_synchronize(self.handle))

    def launch_count(self) -> int:
        return int(lib().fusg_ctx_launch_count(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().fusg_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_contexts = {}


def context(device: Optional[int] = None) -> Context:
    if device is None:
        device = torch.cuda.current_device() if torch is not None and torch.cuda.is_available() else 0
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


def _on_device(a, ctx: Context):
    """complex128 contiguous CUDA tensor view of a field (copies host arrays)."""
    if torch is None:
        raise _lib.FusgError("torch is required for device buffers")
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128))
    if not isinstance(a, torch.Tensor):
        a = torch.as_tensor(np.asarray(a, dtype=np.complex128))
    if a.dtype != torch.complex128:
        a = a.to(torch.complex128)
    return a.to(f"cuda:{ctx.device}").contiguous().reshape(-1)


def _sync_torch_to(ctx: Context):
    """Order the library's stream after torch's current stream (inputs produced by torch)."""
    torch.cuda.current_stream(ctx.device).synchronize()


# ------------------------------------------------------------------------ L1 types
@dataclass
class Medium:
    """include/fus/medium.hpp:12-23"""
    name: str
    rho0: float
    c0: float
    beta: float
    alpha0: float
    eta: float

    def c(self):
        return _lib.MediumC(self.rho0, self.c0, self.beta, self.alpha0, self.eta)

    def validate(self) -> list:
        """src/medium.cpp:11-23: ValueError for impossible values, warnings otherwise."""
        for key, bad, what in (("rho0", self.rho0 <= 0.0, "must be positive"), ("c0", self.c0 <= 0.0, "must be positive"),
                               ("beta", self.beta < 0.0, "must be non-negative"),
                               ("alpha0", self.alpha0 < 0.0, "must be non-negative")):
            if bad:
                raise ValueError(f"medium '{self.name}': {key} {what}")
        if self.eta < 1.0 or self.eta > 2.0:
            return [f"medium '{self.name}': power-law exponent eta={self.eta:f} is outside the typical range [1, 2]"]
        return []


@dataclass
class Wavenumber:
    """include/fus/medium.hpp:26-30"""
    k: complex
    harmonic: int
    omega: float

    def c(self):
        return _lib.Wave(self.k.real, self.k.imag, self.harmonic, self.omega)


K_DB_PER_NEPER = 8.685889638065035


def medium_preset(name: str) -> Medium:
    """src/medium.cpp:47-52"""
    table = {"water": (1000.0, 1480.0, 3.5, 0.2, 2.0), "liver": (1060.0, 1590.0, 4.4, 90.0, 1.1),
             "kidney": (1050.0, 1570.0, 4.7, 10.0, 1.0)}
    if name not in table:
        raise ValueError(f"unknown medium preset '{name}'")
    return Medium(name, *table[name])


def is_medium_preset(name: str) -> bool:
    return name in ("water", "liver", "kidney")


def load_medium(path: str) -> Medium:
    """src/medium.cpp:58-69: key=value file with name, rho0, c0, beta, alpha0, eta."""
    kv = parse_key_value_file(path)
    m = Medium(require_string(kv, "name", path), require_double(kv, "rho0", path), require_double(kv, "c0", path),
               require_double(kv, "beta", path), require_double(kv, "alpha0", path), require_double(kv, "eta", path))
    import sys as _sys
    for w in m.validate():
        print(f"warning: {w}", file=_sys.stderr)
    return m


def complex_wavenumber(m: Medium, f0: float, n: int) -> Wavenumber:
    """src/medium.cpp:31-45"""
    w = _lib.Wave()
    mc = m.c()
    check(lib().fusg_complex_wavenumber(C.byref(mc), float(f0), int(n), C.byref(w)))
    return Wavenumber(complex(w.k_re, w.k_im), w.harmonic, w.omega)


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

    def c(self) -> _lib.Grid:
        g = _lib.Grid()
        for a in range(3):
            g.lo[a], g.hi[a], g.dims[a] = float(self.lo[a]), float(self.hi[a]), int(self.dims[a])
        g.dx, g.harmonic = float(self.dx), int(self.harmonic)
        return g

    @staticmethod
    def from_c(g: _lib.Grid) -> "VoxelGrid":
        return VoxelGrid(np.array(list(g.lo)), np.array(list(g.hi)), g.dx, tuple(g.dims), g.harmonic)


def same_grid(a: VoxelGrid, b: VoxelGrid) -> bool:
    """src/cascade.cpp:15-17"""
    return tuple(a.dims) == tuple(b.dims) and a.dx == b.dx and bool(np.all(a.lo == b.lo))


def _d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def make_grid(lo, hi, dx: float, harmonic: int, anchor=None) -> VoxelGrid:
    """src/grid.cpp:12-34"""
    g = _lib.Grid()
    anc = _d3(anchor) if anchor is not None else None
    check(lib().fusg_make_grid(_d3(lo), _d3(hi), float(dx), int(harmonic), anc, C.byref(g)))
    return VoxelGrid.from_c(g)


@dataclass
class HarmonicField:
    """include/fus/grid.hpp:57-61; values is a complex128 CUDA tensor (x fastest)."""
    grid: VoxelGrid
    values: "torch.Tensor"
    wavenumber: Wavenumber


def random_vector(n: int, seed: int) -> np.ndarray:
    """Seeded input exactly like tests/acceptance.cpp:30-36 (host)."""
    out = np.empty(2 * n, np.float64)
    check(lib().fusg_random_vector(n, seed, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out.view(np.complex128)


# ------------------------------------------------------------------------ potential
def equivalent_sphere_radius(dx: float) -> float:
    return float(lib().fusg_equivalent_sphere_radius(float(dx)))


def self_weight(k: Wavenumber, dx: float) -> complex:
    """src/potential.cpp:59-70"""
    out = (C.c_double * 2)()
    w = k.c()
    check(lib().fusg_self_weight(C.byref(w), float(dx), out))
    return complex(out[0], out[1])


def green_function(x, y, k: Wavenumber) -> complex:
    """src/potential.cpp:47-53 (scalar helper)"""
    d = np.asarray(x, float) - np.asarray(y, float)
    r = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    if r < 1e-300:
        raise ValueError("green_function: singular at x == y")
    mag = math.exp(-k.k.imag * r) / (4.0 * math.pi * r)
    return complex(mag * math.cos(k.k.real * r), mag * math.sin(k.k.real * r))


def evaluate_potential_at(k: Wavenumber, grid: VoxelGrid, f, points, ctx: Optional["Context"] = None) -> np.ndarray:
    """src/potential.cpp:161-201: the volume potential of f (N complex128, host or device) at
    arbitrary points (M x 3) as a host array of M complex128; on the device, O(N M)."""
    n = grid.count()
    size = f.numel() if torch is not None and isinstance(f, torch.Tensor) else np.size(f)
    if size != n:
        raise ValueError("evaluate_potential_at: field size mismatch")
    ctx = ctx or context()
    fd = _on_device(f, ctx)
    pts = np.ascontiguousarray(np.asarray(points, float).reshape(-1, 3))
    out = np.empty(len(pts), np.complex128)
    g, w = grid.c(), k.c()
    _sync_torch_to(ctx)
    check(lib().fusg_evaluate_potential_at(ctx.handle, C.byref(g), C.byref(w), fd.data_ptr(),
                                           pts.ctypes.data, len(pts), out.ctypes.data))
    return out


def direct_potential_oracle(k: Wavenumber, grid: VoxelGrid, f, ctx: Optional["Context"] = None) -> np.ndarray:
    """src/potential.cpp:203-238: the O(N^2) quadrature at every voxel centre (guarded to 1e5
    voxels), run on the device through the off-grid kernel (the coincident point takes the
    self term)."""
    if grid.count() > 100000:
        raise ValueError("direct_potential_oracle: grid exceeds the 1e5 voxel guard")
    size = f.numel() if torch is not None and isinstance(f, torch.Tensor) else np.size(f)
    if size != grid.count():
        raise ValueError("direct_potential_oracle: field size mismatch")
    ax = [grid.lo[a] + (np.arange(grid.dims[a]) + 0.5) * grid.dx for a in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    pts = np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], 1)
    return evaluate_potential_at(k, grid, f, pts, ctx)


def next_fast_size(n: int) -> int:
    return int(lib().fusg_next_fast_size(int(n)))


class GreenKernel:
    """GreenKernel (include/fus/potential.hpp:28-48): octant spectrum cached on the GPU."""

    def __init__(self, grid: VoxelGrid, k: Wavenumber, pad_small_primes: bool = False,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or context()
        self._grid, self._k = grid, k
        h = C.c_void_p()
        g, w = grid.c(), k.c()
        check(lib().fusg_kernel_create(self.ctx.handle, C.byref(g), C.byref(w),
                                       int(bool(pad_small_primes)), C.byref(h)))
        self.handle = h
        p = (C.c_int32 * 3)()
        check(lib().fusg_kernel_padded(h, p))
        self.padded = tuple(p)

    def grid(self) -> VoxelGrid:
        return self._grid

    def wavenumber(self) -> Wavenumber:
        return self._k

    def device_bytes(self) -> int:
        return int(lib().fusg_kernel_device_bytes(self.handle))

    def apply(self, f, scale: float = 1.0, out=None):
        """u = scale * apply(f) (src/potential.cpp:120-151); f: N complex128 (tensor/array).
        Returns a CUDA tensor; synchronous with respect to torch's current stream."""
        if isinstance(f, HarmonicField):
            return HarmonicField(self._grid, self.apply(f.values, scale), self._k)
        n = self._grid.count()
        if (f.numel() if torch is not None and isinstance(f, torch.Tensor) else np.size(f)) != n:
            raise ValueError("GreenKernel::apply: field size does not match kernel grid")
        fd = _on_device(f, self.ctx)
        if out is not None:
            if (not isinstance(out, torch.Tensor) or out.dtype != torch.complex128 or out.numel() != n
                    or not out.is_contiguous() or out.device != fd.device):
                raise ValueError("GreenKernel::apply: out must be a contiguous complex128 tensor of "
                                 f"{n} elements on {fd.device}")
        u = out if out is not None else torch.empty(n, dtype=torch.complex128, device=fd.device)
        _sync_torch_to(self.ctx)
        check(lib().fusg_kernel_apply(self.handle, fd.data_ptr(), u.data_ptr(), float(scale), None))
        self.ctx.synchronize()
        return u

    def apply_async(self, f_ptr: int, u_ptr: int, scale: float = 1.0, stream: int = 0):
        """Raw device-pointer apply on `stream` (0 = context stream); no synchronisation."""
        check(lib().fusg_kernel_apply(self.handle, f_ptr, u_ptr, float(scale), stream or None))

    def apply_host(self, f: np.ndarray, scale: float = 1.0, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Host-vector drop-in (GreenKernel::apply(const VectorXcd&)): H2D, apply, D2H, chunk-
        pipelined; pageable arrays are staged through the library's pinned ring."""
        f = np.ascontiguousarray(f, np.complex128).reshape(-1)
        if f.size != self._grid.count():
            raise ValueError("GreenKernel::apply: field size does not match kernel grid")
        if out is not None:
            if (not isinstance(out, np.ndarray) or out.dtype != np.complex128 or out.size != f.size
                    or not out.flags.c_contiguous):
                raise ValueError(f"GreenKernel::apply: out must be a contiguous complex128 array of {f.size} elements")
            u = out.reshape(-1)
        else:
            u = np.empty_like(f)
        check(lib().fusg_kernel_apply_host(self.handle, f.ctypes.data, u.ctypes.data, float(scale)))
        return u

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().fusg_kernel_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def static_lengths(conv: bool = False) -> list:
    """Padded lengths with compile-time-planned kernels (x/y passes, or pass C on z)."""
    n = int(lib().fusg_static_lengths(int(conv), None, 0))
    out = (C.c_int32 * n)()
    lib().fusg_static_lengths(int(conv), out, n)
    return list(out)


def padded_dims(grid: VoxelGrid, pad_small_primes: bool = False) -> tuple:
    out = (C.c_int32 * 3)()
    g = grid.c()
    check(lib().fusg_padded_dims(C.byref(g), int(pad_small_primes), out))
    return tuple(out)


# ------------------------------------------------------------------------ transducer
@dataclass
class BowlTransducer:
    """include/fus/transducer.hpp:15-28"""
    name: str
    f0: float
    focal_length: float
    outer_radius: float
    power: float
    source_points: np.ndarray

    def focus(self):
        return np.array([self.focal_length, 0.0, 0.0])

    def cap_area(self) -> float:
        l, R = self.focal_length, self.outer_radius
        return 2.0 * math.pi * l * (l - math.sqrt(l * l - R * R))

    def rim_plane_x(self) -> float:
        l, R = self.focal_length, self.outer_radius
        return l - math.sqrt(l * l - R * R)

    def _src(self):
        self._pts = np.ascontiguousarray(self.source_points, np.float64)
        return self._pts.ctypes.data_as(C.POINTER(C.c_double)), len(self._pts)

    def c(self) -> _lib.Bowl:
        p, n = self._src()
        return _lib.Bowl(self.f0, self.focal_length, self.outer_radius, self.power, n, p)


def distribute_points(l: float, R: float, n: int) -> np.ndarray:
    """src/transducer.cpp:22-70"""
    out = np.empty(3 * int(n), np.float64)
    check(lib().fusg_distribute_points(float(l), float(R), int(n),
                                       out.ctypes.data_as(C.POINTER(C.c_double))))
    return out.reshape(-1, 3)


def load_transducer(path: str, power: float) -> "BowlTransducer":
    """src/transducer.cpp:94-102: key=value file with name, f0, focal_length, outer_radius, n_points."""
    kv = parse_key_value_file(path)
    return make_bowl(require_string(kv, "name", path), require_double(kv, "f0", path),
                     require_double(kv, "focal_length", path), require_double(kv, "outer_radius", path), power,
                     int(require_double(kv, "n_points", path)))


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


def unnormalized_field(t: BowlTransducer, pts, k: Wavenumber, amp: Optional[float] = None,
                       ctx: Optional[Context] = None):
    """src/transducer.cpp:123-132; returns a CUDA tensor."""
    ctx = ctx or context()
    if amp is None:
        amp = t.cap_area() / float(len(t.source_points))
    p = torch.as_tensor(np.ascontiguousarray(np.asarray(pts, float).reshape(-1, 3))).to(f"cuda:{ctx.device}")
    out = torch.empty(p.shape[0], dtype=torch.complex128, device=p.device)
    sp, n = t._src()
    _sync_torch_to(ctx)
    check(lib().fusg_monopole_points(ctx.handle, sp, n, p.data_ptr(), p.shape[0], k.k.real,
                                     k.k.imag, float(amp), out.data_ptr(), None))
    return out


def radiated_power(t: BowlTransducer, m: Medium, k: Wavenumber, amplitude_scale: float,
                   n_r: int = 384, n_theta: int = 256, ctx: Optional[Context] = None) -> float:
    """src/transducer.cpp:134-155"""
    ctx = ctx or context()
    amp = amplitude_scale * t.cap_area() / float(len(t.source_points))
    sp, n = t._src()
    out = C.c_double()
    check(lib().fusg_radiated_power(ctx.handle, sp, n, t.rim_plane_x(), t.outer_radius, k.k.real,
                                    k.k.imag, amp, m.rho0, m.c0, int(n_r), int(n_theta),
                                    C.byref(out)))
    return out.value


def power_scale_factor(t: BowlTransducer, m: Medium, k: Wavenumber) -> float:
    """src/transducer.cpp:157-163"""
    if t.power == 0.0:
        return 0.0
    pw = radiated_power(t, m, k, 1.0)
    if pw <= 0.0:
        raise RuntimeError("power normalization: degenerate field, Pi(p) = 0")
    return math.sqrt(t.power / pw)


def evaluate_first_harmonic(t: BowlTransducer, m: Medium, grid: VoxelGrid, amplitude_scale: float,
                            ctx: Optional[Context] = None) -> HarmonicField:
    """src/transducer.cpp:179-196"""
    ctx = ctx or context()
    k1 = complex_wavenumber(m, t.f0, 1)
    amp = amplitude_scale * t.cap_area() / float(len(t.source_points))
    out = torch.empty(grid.count(), dtype=torch.complex128, device=f"cuda:{ctx.device}")
    sp, n = t._src()
    g = grid.c()
    _sync_torch_to(ctx)
    check(lib().fusg_monopole_grid(ctx.handle, sp, n, C.byref(g), k1.k.real, k1.k.imag, amp,
                                   out.data_ptr(), None))
    return HarmonicField(grid, out, k1)


def evaluate_first_harmonic_zslab(t: BowlTransducer, m: Medium, grid: VoxelGrid, amplitude_scale: float,
                                  z0: int, nz: int, ctx: Optional[Context] = None):
    """Planes [z0, z0 + nz) of evaluate_first_harmonic (src/transducer.cpp:179-196), bitwise the
    same values: the multi-GPU incident field shards by z-planes with no collective (each rank
    evaluates its own slab).  Returns a CUDA complex128 tensor of Nx*Ny*nz."""
    ctx = ctx or context()
    k1 = complex_wavenumber(m, t.f0, 1)
    amp = amplitude_scale * t.cap_area() / float(len(t.source_points))
    nx, ny, _ = grid.dims
    out = torch.empty(nx * ny * nz, dtype=torch.complex128, device=f"cuda:{ctx.device}")
    sp, n = t._src()
    g = grid.c()
    _sync_torch_to(ctx)
    check(lib().fusg_monopole_grid_zslab(ctx.handle, sp, n, C.byref(g), int(z0), int(nz), k1.k.real,
                                         k1.k.imag, amp, out.data_ptr() if nz > 0 else None, None))
    return out


def evaluate_source_field(t: BowlTransducer, m: Medium, grid: VoxelGrid):
    """src/transducer.cpp:198-206 -> (field, normalization)"""
    k1 = complex_wavenumber(m, t.f0, 1)
    scale = power_scale_factor(t, m, k1)
    f = evaluate_first_harmonic(t, m, grid, scale)
    return f, (scale if scale > 0.0 else 1.0)


# ------------------------------------------------------------------------ planner
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


def _plan(t, m, d, n_w, n_h, width_scale, single):
    nh = max(int(n_h) - 1, 0)
    grids = (_lib.Grid * max(nh, 1))()
    lo = (C.c_double * (3 * max(nh, 1)))()
    hi = (C.c_double * (3 * max(nh, 1)))()
    ref = _lib.Grid()
    w = C.c_double()
    tb, mc = t.c(), m.c()
    check(lib().fusg_plan_nested_meshes(C.byref(tb), C.byref(mc), float(d), int(n_w), int(n_h),
                                        float(width_scale), int(single), grids, lo, hi,
                                        C.byref(ref), C.byref(w)))
    pgs = [PlannedGrid(i + 2, np.array(lo[3 * i:3 * i + 3]), np.array(hi[3 * i:3 * i + 3]),
                       VoxelGrid.from_c(grids[i])) for i in range(nh)]
    return MeshPlan(pgs, VoxelGrid.from_c(ref), float(d), w.value, t.focus(), int(n_w))


def plan_nested_meshes(t, m, d, n_w, n_harmonics, width_scale=1.0) -> MeshPlan:
    """src/grid.cpp:81-112"""
    return _plan(t, m, d, n_w, n_harmonics, width_scale, False)


def plan_single_mesh(t, m, d, n_w, n_harmonics, width_scale=1.0) -> MeshPlan:
    """src/cascade.cpp:109-118"""
    return _plan(t, m, d, n_w, n_harmonics, width_scale, True)


def interpolate(fld: HarmonicField, target: VoxelGrid, ctx: Optional[Context] = None) -> HarmonicField:
    """src/grid.cpp:141-195"""
    ctx = ctx or context()
    v = _on_device(fld.values, ctx)
    if v.numel() != fld.grid.count():
        raise ValueError("interpolate: field size does not match its grid")
    out = torch.empty(target.count(), dtype=torch.complex128, device=v.device)
    sg, tg = fld.grid.c(), target.c()
    _sync_torch_to(ctx)
    check(lib().fusg_interpolate(ctx.handle, C.byref(sg), v.data_ptr(), C.byref(tg), out.data_ptr(), None))
    ctx.synchronize()
    return HarmonicField(target, out, fld.wavenumber)


# ------------------------------------------------------------------------ cascade
def interpolate_source_planes(src: VoxelGrid, target: VoxelGrid, tz0: int, tnz: int) -> tuple:
    """Source planes (z_lo, z_hi) that target planes [tz0, tz0 + tnz) of interpolate read."""
    lo, hi = C.c_int32(), C.c_int32()
    gs, gt = src.c(), target.c()
    check(lib().fusg_interpolate_source_planes(C.byref(gs), C.byref(gt), int(tz0), int(tnz), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def interpolate_zslab(src: VoxelGrid, f_slab, sz0: int, target: VoxelGrid, tz0: int, tnz: int,
                      ctx: Optional[Context] = None):
    """Target planes [tz0, tz0 + tnz) of interpolate (src/grid.cpp:141-195) from a source z-slab
    f_slab holding planes [sz0, sz0 + len/(Nx Ny)) (halo included): the multi-GPU transfer,
    bitwise the full transfer's planes."""
    ctx = ctx or context()
    fs = _on_device(f_slab, ctx)
    nxs, nys, _ = src.dims
    snz = fs.numel() // (nxs * nys)
    nx, ny, _ = target.dims
    out = torch.empty(nx * ny * tnz, dtype=torch.complex128, device=f"cuda:{ctx.device}")
    gs, gt = src.c(), target.c()
    _sync_torch_to(ctx)
    check(lib().fusg_interpolate_zslab(ctx.handle, C.byref(gs), int(sz0), int(snz), fs.data_ptr(), C.byref(gt),
                                       int(tz0), int(tnz), out.data_ptr() if tnz > 0 else None, None))
    return out


def rhs_source(n: int, lower: Sequence[HarmonicField], m: Medium, omega: float,
               ctx: Optional[Context] = None):
    """src/cascade.cpp:21-40; returns a CUDA tensor."""
    ctx = ctx or context()
    if n < 2:
        raise ValueError("rhs_source: harmonic index must be >= 2")
    if len(lower) < n - 1:
        raise ValueError(f"rhs_source: missing lower harmonics for n = {n}")
    vals = [_on_device(h.values, ctx) for h in lower[: n - 1]]
    count = vals[0].numel()
    if any(v.numel() != count for v in vals):
        raise ValueError("rhs_source: lower harmonics live on different grids")
    ptrs = (C.c_void_p * len(vals))(*[v.data_ptr() for v in vals])
    out = torch.empty(count, dtype=torch.complex128, device=vals[0].device)
    mc = m.c()
    _sync_torch_to(ctx)
    check(lib().fusg_rhs_source(ctx.handle, int(n), ptrs, count, C.byref(mc), float(omega),
                                out.data_ptr(), None))
    ctx.synchronize()
    return out


def rhs_source_full(n: int, fields: Sequence[HarmonicField], m: Medium, omega: float,
                    ctx: Optional[Context] = None):
    """The paper's full quadratic source truncated at M = len(fields):
    coeff * [sum_{m<n} p_m p_{n-m} + 2 sum_{m=n+1}^{M} p_m conj(p_{m-n})]; fields = p_1 .. p_M on
    one grid (fields[n-1], p_n, enters only through p_{2n} conj(p_n) and may be None when
    2n > M). M = n - 1 reproduces rhs_source bit for bit."""
    ctx = ctx or context()
    M = len(fields)
    if n < 2:
        raise ValueError("rhs_source: harmonic index must be >= 2")
    if M < n - 1:
        raise ValueError(f"rhs_source_full: missing lower harmonics for n = {n}")
    vals = [None if fields[i] is None else _on_device(fields[i].values, ctx) for i in range(M)]
    count = next(v for v in vals if v is not None).numel()
    if any(v is not None and v.numel() != count for v in vals):
        raise ValueError("rhs_source_full: harmonics live on different grids")
    ptrs = (C.c_void_p * M)(*[0 if v is None else v.data_ptr() for v in vals])
    out = torch.empty(count, dtype=torch.complex128, device=f"cuda:{ctx.device}")
    mc = m.c()
    _sync_torch_to(ctx)
    check(lib().fusg_rhs_source_full(ctx.handle, int(n), ptrs, int(M), count, C.byref(mc), float(omega),
                                     out.data_ptr(), None))
    ctx.synchronize()
    return out


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
class StageTiming:
    """include/fus/cascade.hpp:25-32 (+ p1_s, rhs_s)"""
    harmonic: int
    voxels: int
    meshing_s: float
    interpolation_s: float
    kernel_s: float
    potential_s: float
    p1_s: float = 0.0
    rhs_s: float = 0.0


@dataclass
class CascadeResult:
    """include/fus/cascade.hpp:34-40"""
    harmonics: List[HarmonicField] = field(default_factory=list)
    timings: List[StageTiming] = field(default_factory=list)
    source_normalization: float = 1.0

    def p(self, n: int) -> HarmonicField:
        return self.harmonics[n - 1]


def run_cascade(cfg: CascadeConfig, ctx: Optional[Context] = None) -> CascadeResult:
    """src/cascade.cpp:42-107, device resident (fusg_run_cascade)."""
    ctx = ctx or context()
    n = int(cfg.n_harmonics)
    if n < 2:
        raise ValueError("run_cascade: n_harmonics must be >= 2")
    grids = [cfg.plan.for_harmonic(i).grid for i in range(2, n + 1)]
    cg = (_lib.Grid * len(grids))(*[g.c() for g in grids])
    dev = f"cuda:{ctx.device}"
    outs = [torch.empty(grids[max(i - 1, 0)].count(), dtype=torch.complex128, device=dev)
            for i in range(n)]
    ptrs = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    rows = (_lib.StageTiming * (n - 1))()
    norm = C.c_double()
    desc = _lib.CascadeDesc(cfg.medium.c(), cfg.transducer.c(), cg, n,
                            int(cfg.recompute_p1_each_grid), int(cfg.pad_small_primes))
    _sync_torch_to(ctx)
    check(lib().fusg_run_cascade(ctx.handle, C.byref(desc), ptrs, rows, C.byref(norm)))
    res = CascadeResult(source_normalization=norm.value)
    for i in range(n):
        g = grids[max(i - 1, 0)]
        k = complex_wavenumber(cfg.medium, cfg.transducer.f0, i + 1)
        res.harmonics.append(HarmonicField(g, outs[i], k))
    for r in rows:
        res.timings.append(StageTiming(r.harmonic, int(r.voxels), r.meshing_s, r.interpolation_s,
                                       r.kernel_s, r.potential_s, r.p1_s, r.rhs_s))
    return res


def _zsplit(n: int, G: int):
    """Ragged z-slabs [(z0, nz)] of n planes over G ranks (the first n mod G take one more)."""
    out, z0 = [], 0
    for r in range(G):
        nz = n // G + (1 if r < n % G else 0)
        out.append((z0, nz))
        z0 += nz
    return out


def run_cascade_zslab_loopback(cfg: CascadeConfig, nranks: int, ctx: Optional[Context] = None,
                               transport: str = "auto") -> CascadeResult:
    """The cascade of run_cascade (src/cascade.cpp:42-107) decomposed into z-slabs as a multi-GPU
    run would be, all ranks in this process on one GPU: the incident field per
    slab (no collective), each lower harmonic brought onto the next grid per target slab from
    its source slab plus the halo planes a neighbour would send (fusg_interpolate_zslab), the
    source term per slab, and the apply through the slab-sharded operator (fused peer-store
    transposes where the padded x / y lengths have transposing warp kernels, else NCCL; "auto").
    The result must equal run_cascade's bit for bit."""
    ctx = ctx or context()
    n = int(cfg.n_harmonics)
    if n < 2:
        raise ValueError("run_cascade: n_harmonics must be >= 2")
    t, med = cfg.transducer, cfg.medium
    grid_of = lambda i: cfg.plan.for_harmonic(max(i, 2)).grid  # p1 lives on D_2's grid
    k1 = complex_wavenumber(med, t.f0, 1)
    scale = power_scale_factor(t, med, k1)
    norm = scale if scale > 0.0 else 1.0
    g1 = grid_of(1)
    fields = [torch.cat([evaluate_first_harmonic_zslab(t, med, g1, scale, z0, nz, ctx)
                         for z0, nz in _zsplit(g1.dims[2], nranks)])]
    res = CascadeResult(source_normalization=norm)
    res.harmonics.append(HarmonicField(g1, fields[0], k1))

    class _Slab:  # rhs_source only reads .values
        def __init__(self, v):
            self.values = v

    for i in range(2, n + 1):
        gi = grid_of(i)
        ki = complex_wavenumber(med, t.f0, i)
        plane = gi.dims[0] * gi.dims[1]
        rhs_slabs = []
        for z0, nz in _zsplit(gi.dims[2], nranks):
            lower = []
            for m in range(1, i):
                gm, pm = grid_of(m), fields[m - 1]
                if same_grid(gm, gi):
                    lower.append(_Slab(pm[z0 * plane:(z0 + nz) * plane]))
                    continue
                if cfg.recompute_p1_each_grid and m == 1:
                    lower.append(_Slab(evaluate_first_harmonic_zslab(t, med, gi, scale, z0, nz, ctx)))
                    continue
                if nz == 0:
                    lower.append(_Slab(torch.empty(0, dtype=torch.complex128, device=pm.device)))
                    continue
                lo, hi = interpolate_source_planes(gm, gi, z0, nz)
                pl = gm.dims[0] * gm.dims[1]
                lower.append(_Slab(interpolate_zslab(gm, pm[lo * pl:(hi + 1) * pl], lo, gi, z0, nz, ctx)))
            rhs_slabs.append(rhs_source(i, lower, med, ki.omega, ctx) if nz > 0 else
                             torch.empty(0, dtype=torch.complex128, device=fields[0].device))
        f = torch.cat(rhs_slabs)
        gk = VoxelGrid(gi.lo, gi.hi, gi.dx, gi.dims, i)
        tr = transport
        if tr == "auto":
            px, py = padded_dims(gk)[:2]
            warp = {256, 512, 768, 1024, 1536}
            tr = "p2p" if px in warp and py in warp else "nccl"
        u = apply_slab_loopback(gk, ki, f, nranks, -1.0, ctx, tr)
        fields.append(u)
        res.harmonics.append(HarmonicField(gi, u, ki))
    return res


# ------------------------------------------------------------------------ VIE mode
# SURVEY.md 8(f) rank 2 (include/fus/vie.hpp, src/vie.cpp): heterogeneous media by a volume
# integral equation solved with restarted GMRES, everything device resident.
class ConvergenceError(RuntimeError):
    """fus::ConvergenceError (include/fus/vie.hpp:60-65): carries the residual history."""

    def __init__(self, what: str, residual_history):
        super().__init__(what)
        self.residual_history = list(residual_history)


@dataclass
class MediumMap:
    """include/fus/vie.hpp:17-33: per-voxel sound speed and nonlinearity on a grid."""
    grid: VoxelGrid
    c: np.ndarray
    beta: np.ndarray
    background: Medium

    def _packed(self, ctx) -> "torch.Tensor":  # (c, beta) interleaved, as one complex field
        return _on_device(np.ascontiguousarray(self.c, float) + 1j * np.ascontiguousarray(self.beta, float), ctx)

    def wavenumber_contrast(self, f0: float, n: int, ctx: Optional[Context] = None):
        """src/vie.cpp:11-23 on the device; returns a CUDA tensor of N complex128."""
        ctx = ctx or context()
        m = self._packed(ctx)
        out = torch.empty_like(m)
        bg = self.background.c()
        _sync_torch_to(ctx)
        check(lib().fusg_vie_contrast(ctx.handle, m.data_ptr(), m.numel(), C.byref(bg), float(f0), int(n),
                                      out.data_ptr(), None))
        ctx.synchronize()
        return out

    def contrast_support(self, tol: float = 0.0) -> np.ndarray:
        """src/vie.cpp:25-31"""
        return np.nonzero((np.abs(self.c - self.background.c0) > tol) |
                          (np.abs(self.beta - self.background.beta) > tol))[0]

    def is_homogeneous(self) -> bool:
        return self.contrast_support().size == 0

    def resample(self, target: VoxelGrid, ctx: Optional[Context] = None) -> "MediumMap":
        """src/vie.cpp:35-54: one trilinear pass over (c, beta) packed as a complex field."""
        ctx = ctx or context()
        r = interpolate(HarmonicField(self.grid, self._packed(ctx), None), target, ctx).values.cpu().numpy()
        return MediumMap(target, r.real.copy(), r.imag.copy(), self.background)

    def raster(self) -> np.ndarray:
        """Interleaved (c, beta) doubles, x fastest (the C-ABI map layout)."""
        out = np.empty(2 * self.c.size)
        out[0::2], out[1::2] = self.c, self.beta
        return out


def homogeneous_map(grid: VoxelGrid, background: Medium) -> MediumMap:
    """src/vie.cpp:56-63"""
    n = grid.count()
    return MediumMap(grid, np.full(n, background.c0), np.full(n, background.beta), background)


def slab_map(grid: VoxelGrid, background: Medium, inclusion: Medium, x_center: float,
             thickness: float) -> MediumMap:
    """src/vie.cpp:65-81: the inclusion on voxels whose centre x lies in the closed slab."""
    m = homogeneous_map(grid, background)
    x0, x1 = x_center - thickness / 2.0, x_center + thickness / 2.0
    xs = np.array([grid.center(ix, 0, 0)[0] for ix in range(grid.dims[0])])
    inside = np.broadcast_to(((xs >= x0) & (xs <= x1))[None, None, :],
                             (grid.dims[2], grid.dims[1], grid.dims[0])).reshape(-1)
    m.c[inside] = inclusion.c0
    m.beta[inside] = inclusion.beta
    return m


@dataclass
class VieSolution:
    field: "torch.Tensor"
    residual_history: list
    iterations: int = 0


@dataclass
class VieConfig:
    tol: float = 1e-6
    max_iter: int = 200
    restart: int = 30


def vie_operator_apply(fld, contrast, kernel: "GreenKernel"):
    """src/vie.cpp:133-139: p - V_kbar[(k^2 - kbar^2) p]; returns a CUDA tensor."""
    n = kernel._grid.count()
    p, c = _on_device(fld, kernel.ctx), _on_device(contrast, kernel.ctx)
    if p.numel() != n or c.numel() != n:
        raise ValueError("vie_operator_apply: grid mismatch")
    out = torch.empty_like(p)
    _sync_torch_to(kernel.ctx)
    check(lib().fusg_vie_operator_apply(kernel.handle, c.data_ptr(), p.data_ptr(), out.data_ptr(), None))
    kernel.ctx.synchronize()
    return out


def _gmres_call(fn, args, n_hist):
    hist = (C.c_double * n_hist)()
    hl, it = C.c_int32(), C.c_int32()
    st = fn(*args, hist, n_hist, C.byref(hl), C.byref(it))
    h = [hist[i] for i in range(min(hl.value, n_hist))]
    if st == _lib.FUSG_NOT_CONVERGED:
        raise ConvergenceError(lib().fusg_last_error().decode(errors="replace"), h)
    check(st)
    return h, it.value


def gmres(op, rhs, tol: float, max_iter: int, restart: int = 30, ctx: Optional[Context] = None) -> VieSolution:
    """src/vie.cpp:141-236 on the device with a caller operator op(x) -> A x (CUDA tensors)."""
    ctx = ctx or context()
    b = _on_device(rhs, ctx)
    x = torch.empty_like(b)
    xin = torch.empty_like(b)
    errors = []

    def cb(_user, in_ptr, out_ptr):
        try:
            check(lib().fusg_device_copy(ctx.handle, xin.data_ptr(), in_ptr, 16 * b.numel()))
            y = op(xin)
            y = y.to(device=b.device, dtype=torch.complex128).contiguous()
            torch.cuda.synchronize(b.device)
            check(lib().fusg_device_copy(ctx.handle, out_ptr, y.data_ptr(), 16 * b.numel()))
            return 0
        except Exception as e:  # surfaced after the call
            errors.append(e)
            return _lib.FUSG_RUNTIME

    fn = _lib.OperatorFn(cb)
    _sync_torch_to(ctx)
    try:
        h, it = _gmres_call(lib().fusg_gmres, (ctx.handle, fn, None, b.data_ptr(), b.numel(), float(tol),
                                               int(max_iter), int(restart), x.data_ptr()),
                            int(max_iter) + int(max_iter) // max(1, int(restart)) + 4)
    except Exception:
        if errors:
            raise errors[0]
        raise
    return VieSolution(x, h, it)


def solve_vie(rhs, contrast, kernel: "GreenKernel", tol: float = 1e-6, max_iter: int = 200,
              restart: int = 30) -> VieSolution:
    """src/vie.cpp:238-242: (I - V[contrast .]) p = rhs by restarted GMRES, on the device."""
    ctx = kernel.ctx
    b, c = _on_device(rhs, ctx), _on_device(contrast, ctx)
    if b.numel() != kernel._grid.count() or c.numel() != b.numel():
        raise ValueError("solve_vie: grid mismatch")
    x = torch.empty_like(b)
    _sync_torch_to(ctx)
    h, it = _gmres_call(lib().fusg_solve_vie, (kernel.handle, b.data_ptr(), c.data_ptr(), float(tol), int(max_iter),
                                               int(restart), x.data_ptr()),
                        int(max_iter) + int(max_iter) // max(1, int(restart)) + 4)
    return VieSolution(x, h, it)


def run_cascade_inhomogeneous(cfg: "CascadeConfig", master_map: MediumMap, vie: VieConfig = VieConfig(),
                              ctx: Optional[Context] = None) -> "CascadeResult":
    """src/vie.cpp:244-323, device resident (fusg_run_cascade_inhomogeneous)."""
    ctx = ctx or context()
    n = int(cfg.n_harmonics)
    if n < 1:
        raise ValueError("run_cascade_inhomogeneous: n_harmonics must be >= 1")
    grids = [cfg.plan.for_harmonic(i).grid for i in range(2, max(n, 2) + 1)]
    cg = (_lib.Grid * len(grids))(*[g.c() for g in grids])
    dev = f"cuda:{ctx.device}"
    outs = [torch.empty(grids[max(i - 1, 0)].count(), dtype=torch.complex128, device=dev) for i in range(n)]
    ptrs = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    rows = (_lib.StageTiming * max(1, n - 1))()
    norm = C.c_double()
    desc = _lib.CascadeDesc(cfg.medium.c(), cfg.transducer.c(), cg, n, int(cfg.recompute_p1_each_grid),
                            int(cfg.pad_small_primes))
    mg, bg = master_map.grid.c(), master_map.background.c()
    raster = np.ascontiguousarray(master_map.raster())
    vc = _lib.VieConfigC(float(vie.tol), int(vie.max_iter), int(vie.restart))
    _sync_torch_to(ctx)
    check(lib().fusg_run_cascade_inhomogeneous(ctx.handle, C.byref(desc), C.byref(mg), raster.ctypes.data,
                                               C.byref(bg), C.byref(vc), ptrs, rows, C.byref(norm)))
    res = CascadeResult(source_normalization=norm.value)
    for i in range(n):
        k = complex_wavenumber(master_map.background, cfg.transducer.f0, i + 1)
        res.harmonics.append(HarmonicField(grids[max(i - 1, 0)], outs[i], k))
    for r in list(rows)[:n - 1]:
        res.timings.append(StageTiming(r.harmonic, int(r.voxels), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0))
    return res


# ------------------------------------------------------------------------ analysis
# SURVEY.md 8(f) rank 4 and the reference's studies (include/fus/analysis.hpp, src/analysis.cpp):
# the O(N M) off-grid evaluations, sources, transfers and reductions run on the device; the
# profile arithmetic (a few hundred nodes) is host numpy like the reference's.
@dataclass
class OnAxisProfile:
    """include/fus/analysis.hpp:12-16"""
    x: np.ndarray
    p: np.ndarray
    harmonic: int = 1


@dataclass
class ConvergenceRecord:
    """include/fus/analysis.hpp:18-23"""
    harmonic: int
    control: str
    value: float
    error_percent: float


@dataclass
class QuadratureStudy:
    records: List[ConvergenceRecord] = field(default_factory=list)
    slope: float = 0.0


def _axis_weights(lo: float, dx: float, n: int):  # src/analysis.cpp:13-23
    q = (0.0 - lo) / dx - 0.5
    j0 = int(math.floor(q))
    j0 = 0 if j0 < 0 else j0
    if j0 > n - 2:
        j0 = max(0, n - 2)
    t = q - j0
    t = 0.0 if t < 0.0 else t
    if t > 1.0:
        t = 1.0 if n > 1 else 0.0
    return j0, t


def extract_on_axis(fld: HarmonicField) -> OnAxisProfile:
    """src/analysis.cpp:49-68: the two straddling columns in y and z with linear weights."""
    g = fld.grid
    jy, ty = _axis_weights(g.lo[1], g.dx, g.dims[1])
    jz, tz = _axis_weights(g.lo[2], g.dx, g.dims[2])
    jy1, jz1 = min(jy + 1, g.dims[1] - 1), min(jz + 1, g.dims[2] - 1)
    v = fld.values.reshape(g.dims[2], g.dims[1], g.dims[0]) if torch is not None and isinstance(
        fld.values, torch.Tensor) else np.asarray(fld.values).reshape(g.dims[2], g.dims[1], g.dims[0])
    rows = [v[jz, jy], v[jz, jy1], v[jz1, jy], v[jz1, jy1]]
    rows = [r.cpu().numpy() if hasattr(r, "cpu") else np.asarray(r) for r in rows]
    x = np.array([g.lo[0] + (ix + 0.5) * g.dx for ix in range(g.dims[0])])
    p = ((1.0 - ty) * (1.0 - tz) * rows[0] + ty * (1.0 - tz) * rows[1] + (1.0 - ty) * tz * rows[2] +
         ty * tz * rows[3])
    h = fld.wavenumber.harmonic if fld.wavenumber is not None else 1
    return OnAxisProfile(x, p, h)


def resample_profile(prof: OnAxisProfile, nodes) -> np.ndarray:
    """src/analysis.cpp:27-45 (linear, clamped at the ends)."""
    px, pp = prof.x, prof.p
    out = np.empty(len(nodes), np.complex128)
    for i, xv in enumerate(nodes):
        if xv <= px[0]:
            out[i] = pp[0]
        elif xv >= px[-1]:
            out[i] = pp[-1]
        else:
            j = int((xv - px[0]) / (px[1] - px[0]))
            while j + 1 < len(px) and px[j + 1] < xv:
                j += 1
            while j > 0 and px[j] > xv:
                j -= 1
            t = (xv - px[j]) / (px[j + 1] - px[j])
            out[i] = (1.0 - t) * pp[j] + t * pp[j + 1]
    return out


def on_axis_error(p: OnAxisProfile, p_ref: OnAxisProfile, normalizer: OnAxisProfile) -> float:
    """src/analysis.cpp:70-78: 100 ||p - p_ref|| / ||normalizer|| on the reference nodes."""
    a = resample_profile(p, p_ref.x)
    denom = float(np.linalg.norm(resample_profile(normalizer, p_ref.x)))
    if denom == 0.0:
        raise ValueError("on_axis_error: normalizer has zero norm")
    return 100.0 * float(np.linalg.norm(a - p_ref.p)) / denom


def localisedness_map(fld: HarmonicField, ctx: Optional[Context] = None):
    """src/analysis.cpp:80-90 on the device; returns a CUDA float64 tensor."""
    ctx = ctx or context()
    v = _on_device(fld.values, ctx)
    q = torch.empty(v.numel(), dtype=torch.float64, device=v.device)
    _sync_torch_to(ctx)
    check(lib().fusg_localisedness_map(ctx.handle, v.data_ptr(), v.numel(), q.data_ptr()))
    return q


def shrink_domain_by_threshold(fld: HarmonicField, q0: float, ctx: Optional[Context] = None):
    """src/grid.cpp:114-139 on the device -> (lo, hi) of the tightest box holding
    |f| >= max|f| 10^q0."""
    ctx = ctx or context()
    v = _on_device(fld.values, ctx)
    g = fld.grid.c()
    lo, hi, m = (C.c_int32 * 3)(), (C.c_int32 * 3)(), C.c_double()
    _sync_torch_to(ctx)
    check(lib().fusg_field_threshold_box(ctx.handle, C.byref(g), v.data_ptr(), float(q0), lo, hi, C.byref(m)))
    gl = np.asarray(fld.grid.lo, float)
    return gl + np.array(lo[:]) * fld.grid.dx, gl + (np.array(hi[:]) + 1) * fld.grid.dx


def error_trend_diagnostic(p_i: OnAxisProfile, p1: OnAxisProfile, q0: float) -> float:
    """src/analysis.cpp:243-246"""
    return 10.0 * (np.linalg.norm(resample_profile(p_i, p1.x)) / np.linalg.norm(p1.p)) * math.sqrt(abs(q0))


def _axis_nodes(x):
    return np.stack([x, np.zeros_like(x), np.zeros_like(x)], 1)


def quadrature_convergence_study(t: BowlTransducer, m: Medium, domain_lo, domain_hi, n_w_values, n_w_ref: int,
                                 ctx: Optional[Context] = None) -> QuadratureStudy:
    """src/analysis.cpp:92-162: p2 at each n_w evaluated at the n_w_ref solution's axis nodes
    through the potential representation (the reference's criterion 1), on the device."""
    ctx = ctx or context()
    for nw in n_w_values:
        if nw >= n_w_ref:
            raise ValueError("quadrature_convergence_study: n_w_ref must exceed all n_w")
    lambda1 = m.c0 / t.f0
    k1, k2 = complex_wavenumber(m, t.f0, 1), complex_wavenumber(m, t.f0, 2)
    scale = power_scale_factor(t, m, k1)

    def source(nw):
        grid = make_grid(domain_lo, domain_hi, lambda1 / (2.0 * nw), 2)
        p1 = evaluate_first_harmonic(t, m, grid, scale, ctx)
        return grid, rhs_source(2, [p1], m, k2.omega, ctx)

    g, f = source(n_w_ref)
    ref_x = np.array([g.lo[0] + (ix + 0.5) * g.dx for ix in range(g.dims[0])])
    nodes = _axis_nodes(ref_x)
    ref = OnAxisProfile(ref_x, -evaluate_potential_at(k2, g, f, nodes, ctx), 2)
    study = QuadratureStudy()
    sx = sy = sxx = sxy = 0.0
    fitted = 0
    for nw in n_w_values:
        g, f = source(nw)
        prof = OnAxisProfile(ref_x, -evaluate_potential_at(k2, g, f, nodes, ctx), 2)
        err = on_axis_error(prof, ref, ref)
        study.records.append(ConvergenceRecord(2, "n_w", float(nw), err))
        if err > 0.0:
            lx, ly = math.log(float(nw)), math.log(err)
            sx, sy, sxx, sxy = sx + lx, sy + ly, sxx + lx * lx, sxy + lx * ly
            fitted += 1
    if fitted >= 2:
        study.slope = (fitted * sxy - sx * sy) / (fitted * sxx - sx * sx)
    return study


def plan_full_domain(t: BowlTransducer, m: Medium, d: float, n_w: int, n_harmonics: int,
                     width_scale: float = 1.0) -> "MeshPlan":
    """src/analysis.cpp:164-174: every harmonic keeps the D_2 domain at its own resolution."""
    plan = plan_nested_meshes(t, m, d, n_w, n_harmonics, width_scale)
    d2lo, d2hi = np.array(plan.grids[0].domain_lo, float), np.array(plan.grids[0].domain_hi, float)
    lambda1 = m.c0 / t.f0
    for pg in plan.grids:
        pg.domain_lo, pg.domain_hi = d2lo.copy(), d2hi.copy()
        pg.grid = make_grid(d2lo, d2hi, lambda1 / (pg.harmonic * n_w), pg.harmonic, plan.focus)
    return plan


def domain_shrink_study(cfg: "CascadeConfig", reference: "CascadeResult", levels, q0_mode: bool,
                        ctx: Optional[Context] = None) -> List[ConvergenceRecord]:
    """src/analysis.cpp:176-241 on the device (transfers, sources, off-grid evaluation)."""
    ctx = ctx or context()
    medium, t, plan = cfg.medium, cfg.transducer, cfg.plan
    lambda1 = medium.c0 / t.f0
    focus = np.asarray(plan.focus, float)
    p1_ref = extract_on_axis(reference.p(1))
    records = []
    for i in range(2, cfg.n_harmonics + 1):
        pi_ref = extract_on_axis(reference.p(i))
        full = plan.for_harmonic(i)
        ki = complex_wavenumber(medium, t.f0, i)
        integrand = None
        if q0_mode:
            lower = [reference.p(mm) if _same_grid(reference.p(mm).grid, full.grid)
                     else interpolate(reference.p(mm), full.grid, ctx) for mm in range(1, i)]
            integrand = HarmonicField(full.grid, rhs_source(i, lower, medium, ki.omega, ctx), ki)
        for level in levels:
            if q0_mode:
                lo, hi = shrink_domain_by_threshold(integrand, level, ctx)
            else:
                L = focus[0] - full.domain_lo[0]
                w = full.domain_hi[1]
                lo = np.array([focus[0] - level * L, -level * w, -level * w])
                hi = np.array([full.domain_hi[0], level * w, level * w])
            grid = make_grid(lo, hi, lambda1 / (i * plan.n_w), i, focus)
            lower = [interpolate(reference.p(mm), grid, ctx) for mm in range(1, i)]
            f = rhs_source(i, lower, medium, ki.omega, ctx)
            prof = OnAxisProfile(pi_ref.x, -evaluate_potential_at(ki, grid, f, _axis_nodes(pi_ref.x), ctx), i)
            records.append(ConvergenceRecord(i, "Q0" if q0_mode else "fraction", float(level),
                                             on_axis_error(prof, pi_ref, p1_ref)))
    return records


def _same_grid(a: VoxelGrid, b: VoxelGrid) -> bool:
    return tuple(a.dims) == tuple(b.dims) and np.array_equal(np.asarray(a.lo), np.asarray(b.lo))


# ------------------------------------------------------------------------ file formats
# include/fus/io.hpp contracts (src/io.cpp) and the medium-map rasters (include/fus/vie.hpp:42-46)
def _num(v: float) -> str:  # the reference's std::setprecision(17) general notation
    return format(float(v), ".17g")


def parse_key_value_file(path: str) -> dict:
    """'key = value' lines, '#' comments; RuntimeError with the line number when malformed."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise RuntimeError(f"cannot open config file '{path}'")
    kv = {}
    for n, line in enumerate(lines, 1):
        t = line.strip(" \t\r")
        if not t or t.startswith("#"):
            continue
        if "=" not in t:
            raise RuntimeError(f"{path}:{n}: expected 'key = value'")
        key, value = t.split("=", 1)
        key = key.strip(" \t\r")
        if not key:
            raise RuntimeError(f"{path}:{n}: empty key")
        kv[key] = value.strip(" \t\r")
    return kv


def require_string(kv: dict, key: str, context: str) -> str:
    if key not in kv:
        raise RuntimeError(f"{context}: missing required key '{key}'")
    return kv[key]


def require_double(kv: dict, key: str, context: str) -> float:
    s = require_string(kv, key, context)
    try:
        return float(s)
    except ValueError:
        raise RuntimeError(f"{context}: key '{key}' is not a number: '{s}'")


def write_on_axis_csv(path: str, x, p) -> None:
    with open(path, "w") as out:
        out.write("x_m,re_Pa,im_Pa,abs_Pa\n")
        for xv, pv in zip(np.asarray(x, float), np.asarray(p, complex)):
            out.write(f"{_num(xv)},{_num(pv.real)},{_num(pv.imag)},{_num(abs(pv))}\n")


def write_field_dump(path: str, fld: HarmonicField) -> None:
    v = fld.values.cpu().numpy() if hasattr(fld.values, "cpu") else np.asarray(fld.values)
    np.ascontiguousarray(v, "<c16").tofile(path)
    g, k = fld.grid, fld.wavenumber
    with open(path + ".hdr", "w") as h:
        h.write(f"nx = {g.dims[0]}\nny = {g.dims[1]}\nnz = {g.dims[2]}\ndx = {_num(g.dx)}\n"
                f"origin_x = {_num(g.lo[0])}\norigin_y = {_num(g.lo[1])}\norigin_z = {_num(g.lo[2])}\n"
                f"harmonic = {k.harmonic}\nk_re = {_num(k.k.real)}\nk_im = {_num(k.k.imag)}\n"
                "layout = x_fastest_complex_f64_le\n")


def write_csv(path: str, columns, rows) -> None:
    with open(path, "w") as out:
        out.write(",".join(columns) + "\n")
        for row in rows:
            out.write(",".join(_num(v) for v in row) + "\n")


def load_medium_map(header_path: str, background: Medium) -> MediumMap:
    kv = parse_key_value_file(header_path)
    dims = tuple(int(require_double(kv, a, header_path)) for a in ("nx", "ny", "nz"))
    dx = require_double(kv, "dx", header_path)
    lo = np.array([require_double(kv, f"origin_{a}", header_path) for a in "xyz"])
    raster = os.path.join(os.path.dirname(header_path), require_string(kv, "raster", header_path))
    n = dims[0] * dims[1] * dims[2]
    try:
        data = np.fromfile(raster, "<f8")
    except OSError:
        raise RuntimeError(f"cannot open medium-map raster '{raster}'")
    if data.size < 2 * n:
        raise RuntimeError(f"medium-map raster '{raster}' is truncated")
    g = VoxelGrid(lo, lo + np.array(dims) * dx, dx, dims, 1)
    return MediumMap(g, data[0:2 * n:2].copy(), data[1:2 * n:2].copy(), background)


def write_medium_map(header_path: str, raster_path: str, m: MediumMap) -> None:
    g = m.grid
    with open(header_path, "w") as h:
        h.write(f"nx = {g.dims[0]}\nny = {g.dims[1]}\nnz = {g.dims[2]}\ndx = {_num(g.dx)}\n"
                f"origin_x = {_num(g.lo[0])}\norigin_y = {_num(g.lo[1])}\norigin_z = {_num(g.lo[2])}\n"
                f"raster = {os.path.basename(raster_path)}\n")
    m.raster().astype("<f8").tofile(raster_path)


# ------------------------------------------------------------------------ slab sharding
def slab_range(n: int, nranks: int, rank: int):
    """(begin, count) of rank's share of n (ragged: the first n % nranks ranks take one more)."""
    b, c = C.c_int32(), C.c_int32()
    check(lib().fusg_slab_range(int(n), int(nranks), int(rank), C.byref(b), C.byref(c)))
    return b.value, c.value


def slab_exchange_plan(grid: VoxelGrid, nranks: int, rank: int) -> dict:
    """Per-peer element offsets/counts of the two slab transposes (include/fusg.h)."""
    arrs = {k: np.zeros(nranks, np.int64) for k in ("a_off", "a_cnt", "r_off", "r_cnt")}
    g = grid.c()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    check(lib().fusg_slab_exchange_plan(C.byref(g), int(nranks), int(rank), p(arrs["a_off"]),
                                        p(arrs["a_cnt"]), p(arrs["r_off"]), p(arrs["r_cnt"])))
    return arrs


class SlabKernel:
    """GreenKernel for rank `rank` of an nranks-way z-slab decomposition of the global grid."""

    def __init__(self, grid: VoxelGrid, k: Wavenumber, nranks: int, rank: int,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or context()
        self.grid, self.k, self.nranks, self.rank = grid, k, nranks, rank
        h = C.c_void_p()
        g, w = grid.c(), k.c()
        check(lib().fusg_kernel_create_slab(self.ctx.handle, C.byref(g), C.byref(w), 0, int(nranks),
                                            int(rank), C.byref(h)))
        self.handle = h
        v = [C.c_int32() for _ in range(4)]
        check(lib().fusg_kernel_slab(h, *[C.byref(x) for x in v]))
        self.z0, self.nz, self.x0, self.nx = (x.value for x in v)
        kf0, knf = C.c_int32(), C.c_int32()
        check(lib().fusg_kernel_octant_rows(h, C.byref(kf0), C.byref(knf)))
        self.octant_rows = (kf0.value, knf.value)  # folded kx rows of K^ held by this rank

    def slab_count(self) -> int:
        return self.nz * int(self.grid.dims[1]) * int(self.grid.dims[0])

    def apply(self, f_slab, scale: float = 1.0):
        """This rank's apply over NCCL (every rank calls it); f_slab: [nz][Ny][Nx] on device."""
        u = torch.empty_like(f_slab)
        _sync_torch_to(self.ctx)
        check(lib().fusg_kernel_apply_slab(self.handle, f_slab.data_ptr(), u.data_ptr(), float(scale), None))
        self.ctx.synchronize()
        return u

    def ipc_handles(self) -> bytes:
        """This rank's CUDA IPC handles (x-slab, A slab): 128 bytes to all-gather."""
        buf = (C.c_uint8 * 128)()
        check(lib().fusg_kernel_slab_ipc_handles(self.handle, buf))
        return bytes(buf)

    def attach_peers(self, handles: bytes):
        """Map every rank's buffers (handles: all ranks' ipc_handles() concatenated in rank
        order) for the fused peer-memory transposes."""
        if len(handles) != 128 * self.nranks:
            raise ValueError("attach_peers: need 128 bytes per rank")
        buf = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
        check(lib().fusg_kernel_slab_attach_peers(self.handle, buf))

    def apply_p2p(self, f_slab, scale: float = 1.0):
        """This rank's apply with the transposes fused into passes A and D (peer stores over
        NVLink); every rank calls it."""
        u = torch.empty_like(f_slab)
        _sync_torch_to(self.ctx)
        check(lib().fusg_kernel_apply_slab_p2p(self.handle, f_slab.data_ptr(), u.data_ptr(), float(scale), None))
        self.ctx.synchronize()
        return u

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().fusg_kernel_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def attach_nccl(ctx: Context, nranks: int, rank: int, unique_id: bytes):
    """Create this context's NCCL communicator (unique_id from nccl_unique_id() on rank 0)."""
    buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
    check(lib().fusg_ctx_attach_nccl(ctx.handle, int(nranks), int(rank), buf))


def slab_peer_plan(global_grid: VoxelGrid, nranks: int, rank: int) -> dict:
    """Peer-store plan of the fused transposes (fusg_slab_peer_plan): per peer q, the first
    owned key and the flat-index offset / outer stride of rank `rank`'s stores into q."""
    arrs = {n: np.zeros(nranks, np.int64) for n in ("a_begin", "a_off", "a_sk", "d_begin", "d_off", "d_sk")}
    g = global_grid.c()
    ptrs = [a.ctypes.data_as(C.POINTER(C.c_int64)) for a in arrs.values()]
    check(lib().fusg_slab_peer_plan(C.byref(g), int(nranks), int(rank), *ptrs))
    return arrs


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().fusg_nccl_unique_id(buf))
    return bytes(buf)


def apply_slab_loopback(grid: VoxelGrid, k: Wavenumber, f, nranks: int, scale: float = 1.0,
                        ctx: Optional[Context] = None, transport: str = "nccl"):
    """Run an nranks-way slab decomposition of the apply in this process on one GPU and return
    the global u.  transport "nccl": the NCCL path's blocks and kernels, with device copies;
    "p2p": the fused peer-store transposes, with the other in-process ranks as peers."""
    if transport not in ("nccl", "p2p"):
        raise ValueError("apply_slab_loopback: transport is 'nccl' or 'p2p'")
    ctx = ctx or context()
    fd = _on_device(f, ctx)
    ks = [SlabKernel(grid, k, nranks, r, ctx) for r in range(nranks)]
    plane = int(grid.dims[1]) * int(grid.dims[0])
    fs = [fd[kk.z0 * plane:(kk.z0 + kk.nz) * plane].contiguous() for kk in ks]
    us = [torch.empty_like(x) for x in fs]
    hs = (C.c_void_p * nranks)(*[kk.handle.value for kk in ks])
    fp = (C.c_void_p * nranks)(*[x.data_ptr() for x in fs])
    up = (C.c_void_p * nranks)(*[x.data_ptr() for x in us])
    _sync_torch_to(ctx)
    fn = lib().fusg_kernel_apply_slab_loopback_p2p if transport == "p2p" else lib().fusg_kernel_apply_slab_loopback
    check(fn(hs, int(nranks), fp, up, float(scale)))
    return torch.cat(us)
