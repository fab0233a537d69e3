"""CPU oracle for the VIE mode: a function-by-function restatement of
the reference's src/vie.cpp in numpy, on top of fus_oracle (GreenKernel, interpolate,
evaluate_source_field, complex_wavenumber). TEST INFRASTRUCTURE ONLY: only tests/ and bench.py's
CPU legs may import it.

Pinned against the reference's own tests/test_vie.cpp cases in tests/test_oracle_vie.py:
* the VIE operator against the dense assembly of tests/oracles.hpp:47-70;
* GMRES on the random dense system and the shift-operator non-convergence;
* solve_vie against a dense LU solve;
* the first-order Born agreement;
* a homogeneous map reproduces run_cascade.
"""
import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

from oracle import fus_oracle as orc


# --------------------------------------------------------------------------- medium maps
@dataclass
class MediumMap:
    """include/fus/vie.hpp:17-33: per-voxel sound speed and nonlinearity on a grid."""
    grid: orc.VoxelGrid
    c: np.ndarray
    beta: np.ndarray
    background: orc.Medium

    def wavenumber_contrast(self, f0: float, n: int) -> np.ndarray:
        """src/vie.cpp:11-23: k_n(x)^2 - kbar_n^2, k_n(x) = (n omega / c(x), Im kbar_n)."""
        kbar = orc.complex_wavenumber(self.background, f0, n)
        out = np.zeros(self.c.size, np.complex128)
        sel = self.c != self.background.c0
        k = (n * kbar.omega / self.c[sel]) + 1j * kbar.k.imag
        out[sel] = k * k - kbar.k * kbar.k
        return out

    def contrast_support(self, tol: float = 0.0) -> np.ndarray:
        """src/vie.cpp:25-31"""
        return np.nonzero((np.abs(self.c - self.background.c0) > tol) |
                          (np.abs(self.beta - self.background.beta) > tol))[0]

    def is_homogeneous(self) -> bool:
        """src/vie.cpp:33"""
        return self.contrast_support().size == 0

    def resample(self, target: orc.VoxelGrid) -> "MediumMap":
        """src/vie.cpp:35-54: (c, beta) packed as one complex field, one trilinear pass."""
        packed = orc.HarmonicField(self.grid, self.c + 1j * self.beta, None)
        res = orc.interpolate(packed, target)
        return MediumMap(target, res.values.real.copy(), res.values.imag.copy(), self.background)


def homogeneous_map(grid: orc.VoxelGrid, background: orc.Medium) -> MediumMap:
    """src/vie.cpp:56-63"""
    n = grid.count()
    return MediumMap(grid, np.full(n, background.c0), np.full(n, background.beta), background)


def slab_map(grid: orc.VoxelGrid, background: orc.Medium, inclusion: orc.Medium, x_center: float,
             thickness: float) -> MediumMap:
    """src/vie.cpp:65-81: the inclusion where x0 <= x <= x1 (voxel-centre x)."""
    m = homogeneous_map(grid, background)
    x0, x1 = x_center - thickness / 2.0, x_center + thickness / 2.0
    xs = grid.lo[0] + (np.arange(grid.dims[0]) + 0.5) * grid.dx
    inside = (xs >= x0) & (xs <= x1)
    mask = np.broadcast_to(inside[None, None, :], (grid.dims[2], grid.dims[1], grid.dims[0])).reshape(-1)
    m.c[mask] = inclusion.c0
    m.beta[mask] = inclusion.beta
    return m


# --------------------------------------------------------------------------- operator and GMRES
def vie_operator_apply(fld: np.ndarray, contrast: np.ndarray, kernel) -> np.ndarray:
    """src/vie.cpp:133-139: p - V_kbar[(k^2 - kbar^2) p]."""
    if fld.size != contrast.size or fld.size != kernel.grid.count():
        raise ValueError("vie_operator_apply: grid mismatch")
    return fld - kernel.apply(contrast * fld)


@dataclass
class VieSolution:
    field: np.ndarray
    residual_history: List[float] = field(default_factory=list)
    iterations: int = 0


class ConvergenceError(RuntimeError):
    def __init__(self, what, history):
        super().__init__(what)
        self.residual_history = history


def gmres(op, rhs: np.ndarray, tol: float, max_iter: int, restart: int = 30) -> VieSolution:
    """src/vie.cpp:141-236: restarted GMRES, Arnoldi with modified Gram-Schmidt, Givens
    rotations, relative-residual stopping; ConvergenceError past max_iter."""
    if tol <= 0.0:
        raise ValueError("gmres: tol must be positive")
    rhs_norm = float(np.linalg.norm(rhs))
    sol = VieSolution(np.zeros(rhs.size, np.complex128))
    if rhs_norm == 0.0:
        return sol
    total = 0
    while True:
        r = rhs - op(sol.field)
        beta = float(np.linalg.norm(r))
        rel = beta / rhs_norm
        if not sol.residual_history:
            sol.residual_history.append(rel)
        if rel <= tol:
            sol.iterations = total
            return sol
        if total >= max_iter:
            raise ConvergenceError(f"gmres: no convergence within {max_iter} iterations (residual {rel})",
                                   sol.residual_history)
        m = restart
        v = [r / beta]
        h = np.zeros((m + 1, m), np.complex128)
        g = np.zeros(m + 1, np.complex128)
        g[0] = beta
        cs = np.zeros(m, np.complex128)
        sn = np.zeros(m, np.complex128)
        k = 0
        while k < m and total < max_iter:
            w = op(v[k])
            for j in range(k + 1):
                h[j, k] = np.vdot(v[j], w)  # Eigen's dot: conjugate-linear in the first argument
                w = w - h[j, k] * v[j]
            h[k + 1, k] = np.linalg.norm(w)
            for j in range(k):
                tmp = np.conj(cs[j]) * h[j, k] + np.conj(sn[j]) * h[j + 1, k]
                h[j + 1, k] = -sn[j] * h[j, k] + cs[j] * h[j + 1, k]
                h[j, k] = tmp
            denom = math.sqrt(abs(h[k, k]) ** 2 + abs(h[k + 1, k]) ** 2)
            if denom == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = h[k, k] / denom, h[k + 1, k] / denom
            h[k, k] = np.conj(cs[k]) * h[k, k] + np.conj(sn[k]) * h[k + 1, k]
            h[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = np.conj(cs[k]) * g[k]
            rel = abs(g[k + 1]) / rhs_norm
            sol.residual_history.append(rel)
            # (src/vie.cpp:188,213-221: the two early exits do ++k but not ++total_iters)
            if rel <= tol:
                k += 1
                break
            wnorm = float(np.linalg.norm(w))
            if wnorm == 0.0:
                k += 1
                break  # invariant subspace reached
            v.append(w / wnorm)
            k += 1
            total += 1
        y = np.zeros(k, np.complex128)
        for i in range(k - 1, -1, -1):
            s = g[i]
            for j in range(i + 1, k):
                s -= h[i, j] * y[j]
            y[i] = s / h[i, i]
        for i in range(k):
            sol.field = sol.field + y[i] * v[i]
        if rel <= tol:
            sol.iterations = total
            return sol


def solve_vie(rhs, contrast, kernel, tol=1e-6, max_iter=200, restart=30) -> VieSolution:
    """src/vie.cpp:238-242"""
    return gmres(lambda p: vie_operator_apply(p, contrast, kernel), rhs, tol, max_iter, restart)


# --------------------------------------------------------------------------- dense checks
def dense_potential_matrix(k: orc.Wavenumber, g: orc.VoxelGrid) -> np.ndarray:
    """tests/oracles.hpp:47-64 (small grids only)."""
    idx = np.arange(g.count())
    ix, iy, iz = idx % g.dims[0], (idx // g.dims[0]) % g.dims[1], idx // (g.dims[0] * g.dims[1])
    x = np.stack([g.lo[0] + (ix + 0.5) * g.dx, g.lo[1] + (iy + 0.5) * g.dx, g.lo[2] + (iz + 0.5) * g.dx], 1)
    n = g.count()
    W = np.empty((n, n), np.complex128)
    for a in range(0, n, 256):  # row blocks keep the pairwise differences small
        d = x[a:a + 256, None, :] - x[None, :, :]
        r = np.sqrt((d * d).sum(-1))
        r[r == 0.0] = 1.0
        W[a:a + 256] = (g.dx ** 3) * np.exp(-k.k.imag * r) / (4.0 * math.pi * r) * np.exp(1j * k.k.real * r)
    np.fill_diagonal(W, orc.self_weight(k, g.dx))
    return W


def dense_vie_matrix(k, g, contrast) -> np.ndarray:
    """tests/oracles.hpp:66-70: I - W diag(contrast)."""
    return np.eye(g.count()) - dense_potential_matrix(k, g) * contrast[None, :]


# --------------------------------------------------------------------------- cascade
@dataclass
class VieConfig:
    tol: float = 1e-6
    max_iter: int = 200
    restart: int = 30


def run_cascade_inhomogeneous(cfg, master_map: MediumMap, vie: VieConfig = VieConfig(), workers: int = 1):
    """src/vie.cpp:244-323: p1 solves the scattering VIE with the transducer field as right-hand
    side; harmonic i solves a VIE whose right-hand side is -beta(x) omega^2 i^2/(2 rho0 c(x)^4)
    times the convolved quadratic products."""
    plan, n = cfg.plan, cfg.n_harmonics
    if n < 1:
        raise ValueError("run_cascade_inhomogeneous: n_harmonics must be >= 1")
    bg = master_map.background
    f0 = cfg.transducer.f0
    res = orc.CascadeResult()
    grid2 = plan.for_harmonic(2).grid
    p1inc, norm = orc.evaluate_source_field(cfg.transducer, bg, grid2)
    res.source_normalization = norm
    map2 = master_map.resample(grid2)
    contrast1 = map2.wavenumber_contrast(f0, 1)
    if not np.any(contrast1):
        p1 = p1inc.values
    else:
        k1 = orc.complex_wavenumber(bg, f0, 1)
        ker1 = orc.GreenKernel(grid2, k1, workers=workers)
        p1 = solve_vie(p1inc.values, contrast1, ker1, vie.tol, vie.max_iter, vie.restart).field
    res.harmonics.append(orc.HarmonicField(grid2, p1, p1inc.wavenumber))
    for i in range(2, n + 1):
        grid = plan.for_harmonic(i).grid
        lower = []
        for mm in range(1, i):
            pm = res.harmonics[mm - 1]
            lower.append(pm if orc.same_grid(pm.grid, grid) else orc.interpolate(pm, grid))
        map_i = map2 if i == 2 else master_map.resample(grid)
        ki = orc.complex_wavenumber(bg, f0, i)
        products = np.zeros(grid.count(), np.complex128)
        for mm in range(1, i):
            products = products + lower[mm - 1].values * lower[i - mm - 1].values
        kernel = orc.GreenKernel(grid, ki, workers=workers)
        conv = kernel.apply(products)
        n2 = float(i) * float(i)
        coeff = map_i.beta * ki.omega * ki.omega * n2 / (2.0 * bg.rho0 * map_i.c ** 4)
        rhs = -coeff * conv
        contrast = map_i.wavenumber_contrast(f0, i)
        if not np.any(contrast):
            pi = rhs
        else:
            pi = solve_vie(rhs, contrast, kernel, vie.tol, vie.max_iter, vie.restart).field
        res.harmonics.append(orc.HarmonicField(grid, pi, ki))
    return res
