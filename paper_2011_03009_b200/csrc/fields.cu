// Incident field (equal-area monopole / Rayleigh-type sum), radiated-power integral,
// Westervelt quadratic source and trilinear nested-grid transfer.
//
//  * monopole sum  (src/transducer.cpp:107-132,179-196): FP64 CUDA-core kernel, one voxel per
//    thread, sources broadcast from shared memory in the reference's summation order.
//  * radiated power (src/transducer.cpp:134-155): per-node |amp S|^2, then a fixed-order
//    two-level reduction (rings in order, then rings summed in order): deterministic.
//  * rhs_source (src/cascade.cpp:21-40) and interpolate (src/grid.cpp:141-195): elementwise
//    and gather kernels written with explicit round-to-nearest intrinsics, so they round
//    exactly like the reference's non-FMA x86-64 build (bit-identical outputs).
#include <algorithm>
#include <climits>
#include <math_constants.h>
#include <cmath>
#include <vector>

#include "internal.hpp"

namespace fusg {

constexpr int kSrcChunk = 512;  // 12 KB of staged sources (+ 32 KB phase table: static smem)

struct GridDev {
  double lo[3];
  double dx;
  int dims[3];
  int z_off = 0;  // z index of plane 0 (a z-slab of a larger grid: monopole_grid_kernel)
};

static GridDev to_dev(const fusg_grid& g) {
  GridDev d;
  for (int a = 0; a < 3; ++a) {
    d.lo[a] = g.lo[a];
    d.dims[a] = g.dims[a];
  }
  d.dx = g.dx;
  return d;
}

// centre coordinate lo + (i + 0.5) dx, rounded like include/fus/grid.hpp:44-46
__device__ __forceinline__ double centre(double lo, int i, double dx) {
  return __dadd_rn(lo, __dmul_rn(double(i) + 0.5, dx));
}

// One monopole term e^{-Im k d}/(4 pi d) e^{i Re k d} accumulated into acc
// (src/transducer.cpp:110-117).  ATT selects the attenuation factor: 0 none (Im k = 0),
// 1 polynomial (host proved Im k * d <= 0.03 everywhere: degree 6, error < 7e-19),
// 2 exp().
//
// Phase: u = d Re k N / (2 pi) turns-of-table; j = rint(u) (magic-number rounding, whose low
// word is the table index mod N), v = u - j exactly, so e^{i Re k d} = T[j] e^{2 pi i v / N}
// with |2 pi v / N| <= pi / N = 1.5e-3: sin to degree 3 (error < 1e-16 relative) and cos to
// degree 4 (< 1e-19).  T[j] = e^{2 pi i j / N} / (4 pi) lives in shared memory.  The rounding of u
// carries the same absolute phase error as any double evaluation of Re k * d (~1e-16 |k d|).
// 1/d: rsqrt.approx (rel. error < 2^-22) refined by one third-order step (error ~ e^3 < 2^-64).
// Together ~31 FP64 instructions per term against ~47 (+36 constant moves) for sincospi.
constexpr double kInv4Pi = 0.0795774715459476678844;  // 1 / (4 pi)
constexpr double kPolyAttMax = 0.03;
constexpr int kPhaseBits = 11;
constexpr int kPhaseN = 1 << kPhaseBits;
constexpr double kTwoPi = 6.283185307179586476925;
constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52
#ifndef FUSG_MONO_F2I
#define FUSG_MONO_F2I 0  // phase rounding by F2I / I2F conversion (1) or the magic-number add (0)
#endif

// table scale: the host passes k1 = Re k * N / (2 pi)
inline double phase_scale(double kre, int bits = kPhaseBits) { return kre * double(1 << bits) / kTwoPi; }

// Phase-table geometry for N = 2^BITS entries.  The other kernels keep 2048 entries in static
// shared memory.  The grid kernel (the Rayleigh p1 sum) reads its table once per term at an
// effectively random index, and a warp's 32 random 16-byte reads cost ~10.4 wavefronts instead of
// 4 (ncu: 6.3-way conflicts, the shared pipe as busy as the FP64 pipe).  FUSG_MONO_REP = 8: the
// table holds 1024 entries, each replicated 8 times at [j][8] (128 KB), and lane L reads copy
// L % 8, so the 8 lanes of a quarter-warp always hit 8 different 16-byte bank groups: exactly 4
// wavefronts per warp.  The residual |2 pi v / N| <= 3.1e-3 keeps sin at degree 3 (error
// < 2.2e-15) and takes cos to degree 4 (< 1.2e-18): one FP64 instruction more per term.
// Measured on cfg4-desk p1: shared wavefronts 44.8e9 -> 19.3e9 and no bank conflicts, but
// 200.8 vs 189.7 ms, the FP64 pipe at 74 % either way: the shared pipe was not the limit, so the
// extra instruction costs time.  Default FUSG_MONO_REP = 1: 4096 entries, one copy (cos to
// degree 2, error < 1.5e-14).
#ifndef FUSG_MONO_REP
#define FUSG_MONO_REP 1
#endif
constexpr int kGridRep = FUSG_MONO_REP;
static_assert(kGridRep == 1 || kGridRep == 8, "phase-table copies: 1 or 8");
constexpr int kGridPhaseBits = kGridRep == 8 ? 10 : 12;
template <int BITS>
struct PhaseSpec {
  static constexpr int N = 1 << BITS;
  static constexpr double PhC = kTwoPi / N;
  static constexpr double S1 = PhC, S3 = -PhC * PhC * PhC / 6.0;
  static constexpr double C2 = -PhC * PhC / 2.0, C4 = PhC * PhC * PhC * PhC / 24.0;
  static constexpr bool kCos2 = BITS >= 12;  // cos to degree 2
};

// REP copies of each entry, stored [j][REP]
template <int BITS = kPhaseBits, int REP = 1>
__device__ __forceinline__ void fill_phase_table(double2* tab) {
  constexpr int N = 1 << BITS;
  for (int e = threadIdx.x; e < N * REP; e += blockDim.x) {
    const int j = e / REP;
    double sn, cs;
    sincospi(2.0 * j / N, &sn, &cs);  // exact argument (power-of-two denominator)
    tab[e] = make_double2(cs * kInv4Pi, sn * kInv4Pi);
  }
}

// ATT 3 tables (monopole_grid_kernel): rows e^{2 pi i j / N} e^{-alpha j} / (4 pi) and the
// coarse factors eh[m] = e^{-alpha N m}, m < n_eh (the host bounds Re k d / (2 pi) N by N n_eh).
constexpr int kEhMax = 512;
template <int BITS = kPhaseBits, int REP = 1>
__device__ __forceinline__ void fill_att_tables(double2* tab, double* eh, double alpha, int n_eh) {
  constexpr int N = 1 << BITS;
  for (int e = threadIdx.x; e < N * REP; e += blockDim.x) {
    const int j = e / REP;
    double sn, cs;
    sincospi(2.0 * j / N, &sn, &cs);
    const double a = exp(-alpha * j) * kInv4Pi;
    tab[e] = make_double2(cs * a, sn * a);
  }
  for (int m = threadIdx.x; m < n_eh; m += blockDim.x) eh[m] = exp(-alpha * double(N) * m);
}

__device__ __forceinline__ double rsqrt_refined(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);  // 1 - x y^2
  const double p = fma(e, 0.375, 0.5);     // y (1 + e/2 + 3e^2/8)
  return fma(y * e, p, y);
}

template <int ATT>
__device__ __forceinline__ double attenuation(double t) {  // e^{-t}, t = Im k * d >= 0
  if constexpr (ATT == 0) {
    return 1.0;
  } else if constexpr (ATT == 1) {
    // degree-6 interpolant of e^{-t} at the Chebyshev nodes of [0, 0.03] (fitted in long
    // double): approximation error < 7e-19 relative, so Horner rounding (~1 ulp) dominates
    double p = 0.001368220431121461;
    p = fma(p, t, -0.00833248285306652);
    p = fma(p, t, 0.04166664928658103);
    p = fma(p, t, -0.16666666648420275);
    p = fma(p, t, 0.4999999999990874);
    p = fma(p, t, -0.9999999999999983);
    return fma(p, t, 1.0);
  } else {
    return exp(-t);
  }
}

// term from the squared distance d2
// SC (scaled coordinates, monopole_grid_kernel): coordinates arrive pre-multiplied by k1, so d2
// is already in table turns squared, u = d, the magnitude 1/d carries a factor 1/k1 the caller
// restores once per voxel, and the coincidence bound is (k1 1e-12)^2 (bits in tiny_bits).
// REP > 1: the table holds REP copies per entry ([j][REP]) and this lane reads copy `rep`
template <int ATT, bool SC = false, int BITS = kPhaseBits, int REP = 1>
__device__ __forceinline__ void monopole_term_d2(double d2, double k1, double kim,
                                                 const double2* __restrict__ tab, double2& acc,
                                                 bool& bad, const double* __restrict__ eh = nullptr,
                                                 long long tiny_bits = 0x3AF357C299A88EA7LL, int rep = 0) {
  // dist < 1e-12 (src/transducer.cpp:112), i.e. d2 < 1e-24: for d2 >= +0 the IEEE order is the
  // integer order of the bit patterns, so the test runs on the integer pipe, exactly
  bad |= __double_as_longlong(d2) < tiny_bits;
  const double ir = rsqrt_refined(d2);
  const double d = d2 * ir;
  const double u = SC ? d : d * k1;
  using PS = PhaseSpec<BITS>;
#if FUSG_MONO_F2I
  // j = rint(u) by conversion (F2I / I2F) instead of the magic-number add and subtract, off the
  // FP64 pipe's add slots; v = u - j is exact either way (Sterbenz), so the terms are identical
  const int ji = __double2int_rn(u);
  const int j = ji & (PS::N - 1);
  const double v = u - double(ji);
  const int jhi = ji >> BITS;
#else
  const double t = u + kRoundMagic;
  const int j = __double2loint(t) & (PS::N - 1);
  const double v = u - (t - kRoundMagic);
  const int jhi = __double2loint(t) >> BITS;
#endif
  const double v2 = v * v;
  const double sn = v * fma(v2, PS::S3, PS::S1);
  const double cs = PS::kCos2 ? fma(v2, PS::C2, 1.0) : fma(v2, fma(v2, PS::C4, PS::C2), 1.0);
  const double2 w = tab[REP == 1 ? j : j * REP + rep];
  double mag;
  if constexpr (ATT == 3) {
    // tabulated attenuation: kim carries alpha = Im k / k1, the table rows already hold
    // e^{-alpha (j mod N)}, eh[m] = e^{-alpha N m}, and e^{-alpha v} = 1 - alpha v to
    // (alpha v)^2 / 2 < 1e-18
    mag = ir * eh[jhi] * fma(-kim, v, 1.0);
  } else {
    mag = ATT == 0 ? ir : ir * attenuation<ATT>(kim * d);
  }
  const double mc = mag * w.x, ms = mag * w.y;
  acc.x = fma(mc, cs, fma(-ms, sn, acc.x));
  acc.y = fma(mc, sn, fma(ms, cs, acc.y));
}

template <int ATT>
__device__ __forceinline__ void monopole_term(double x, double y, double z, double sx, double sy,
                                              double sz, double k1, double kim,
                                              const double2* __restrict__ tab, double2& acc,
                                              bool& bad) {
  const double ddx = x - sx, ddy = y - sy, ddz = z - sz;
  monopole_term_d2<ATT>(fma(ddz, ddz, fma(ddy, ddy, ddx * ddx)), k1, kim, tab, acc, bad);
}

__device__ __forceinline__ void stage_sources(const double* src, int n_src, int base, double* sx,
                                              double* sy, double* sz, double scale = 1.0) {
  for (int j = threadIdx.x; j < kSrcChunk && base + j < n_src; j += blockDim.x) {
    sx[j] = scale * src[3 * (base + j)];
    sy[j] = scale * src[3 * (base + j) + 1];
    sz[j] = scale * src[3 * (base + j) + 2];
  }
}

// kVPT adjacent voxels of one x-row per thread: the (y, z) part of the squared distance is
// shared, the source loads are amortised and the thread carries kVPT independent chains.
#ifndef FUSG_MONO_VPT
#define FUSG_MONO_VPT 4
#endif
#ifndef FUSG_MONO_THREADS
#define FUSG_MONO_THREADS (kGridRep == 8 ? 512 : 256)  // 128 KB table: one CTA of 16 warps per SM
#endif
constexpr int kVPT = FUSG_MONO_VPT;
#ifndef FUSG_MONO_MINB
#define FUSG_MONO_MINB 1  // CTAs per SM the grid kernel's register budget targets (4: 64 registers, measured equal: FP64-bound)
#endif

template <int ATT>
__global__ void __launch_bounds__(FUSG_MONO_THREADS, FUSG_MONO_MINB) monopole_grid_kernel(const double* __restrict__ src, int n_src,
                                                            GridDev g, double k1, double kim,
                                                            double amp, double2* __restrict__ out,
                                                            int* flag, int n_eh = 0) {
  // coordinates scaled by k1 (distances in table turns, SC terms); kim arrives as Im k / k1
  __shared__ double sx[kSrcChunk], sy[kSrcChunk], sz[kSrcChunk];
  extern __shared__ double2 dyn_tab[];  // phase table (2^kGridPhaseBits) + ATT 3 coarse table
  double2* const tab = dyn_tab;
  double* const eh = reinterpret_cast<double*>(dyn_tab + (kGridRep << kGridPhaseBits));
  // visible after the first barrier of the source loop
  if constexpr (ATT == 3) fill_att_tables<kGridPhaseBits, kGridRep>(tab, eh, kim, n_eh);
  else fill_phase_table<kGridPhaseBits, kGridRep>(tab);
  const int rep = threadIdx.x & (kGridRep - 1);  // this lane's table copy
  const int row_threads = (g.dims[0] + kVPT - 1) / kVPT;
  const int64_t count = int64_t(row_threads) * g.dims[1] * g.dims[2];
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = idx < count;
  int ix0 = 0, nv = 0;
  int64_t row = 0;
  double x[kVPT], y = 0, z = 0;
  if (active) {
    ix0 = int(idx % row_threads) * kVPT;
    row = idx / row_threads;
    nv = min(kVPT, g.dims[0] - ix0);
    y = k1 * centre(g.lo[1], int(row % g.dims[1]), g.dx);
    z = k1 * centre(g.lo[2], int(row / g.dims[1]) + g.z_off, g.dx);
  }
#pragma unroll
  for (int v = 0; v < kVPT; ++v) x[v] = k1 * centre(g.lo[0], ix0 + min(v, max(nv - 1, 0)), g.dx);  // tail: repeat the last voxel
  const long long tiny_bits = __double_as_longlong(k1 * 1e-12 * (k1 * 1e-12));
  double2 acc[kVPT];
#pragma unroll
  for (int v = 0; v < kVPT; ++v) acc[v] = make_double2(0.0, 0.0);
  bool bad = false;
  // The bowl's points come ring by ring (distribute_points), and every point of a ring has the
  // same x (one polar angle): the x part (x_v - s_x)^2 of the squared distance is recomputed only
  // when s_x changes (a warp-uniform branch), one FP64 subtraction per term fewer.
  double px[kVPT];
  double s_prev = __longlong_as_double(0x7ff8000000000000LL);  // NaN: the first source differs
  for (int base = 0; base < n_src; base += kSrcChunk) {
    __syncthreads();
    stage_sources(src, n_src, base, sx, sy, sz, k1);
    __syncthreads();
    if (active) {
      const int n = min(kSrcChunk, n_src - base);
      #pragma unroll 2
      for (int j = 0; j < n; ++j) {
        const double s0 = sx[j];
        if (s0 != s_prev) {
          s_prev = s0;
#pragma unroll
          for (int v = 0; v < kVPT; ++v) {
            const double ddx = x[v] - s0;
            px[v] = ddx * ddx;
          }
        }
        const double ddy = y - sy[j], ddz = z - sz[j];
        const double q = fma(ddz, ddz, ddy * ddy);
#pragma unroll
        for (int v = 0; v < kVPT; ++v)
          monopole_term_d2<ATT, true, kGridPhaseBits, kGridRep>(px[v] + q, k1, kim, tab, acc[v], bad, eh, tiny_bits, rep);
      }
    }
  }
  if (active) {
    if (bad) atomicExch(flag, 1);
    double2* o = out + row * g.dims[0] + ix0;
    const double a = amp * k1;  // the terms' 1/d is in table turns: 1/d = k1 / d'
#pragma unroll
    for (int v = 0; v < kVPT; ++v)
      if (v < nv) o[v] = make_double2(a * acc[v].x, a * acc[v].y);
  }
}

template <int ATT>
__global__ void __launch_bounds__(256) monopole_points_kernel(const double* __restrict__ src,
                                                              int n_src,
                                                              const double* __restrict__ pts,
                                                              int64_t n_pts, double k1, double kim,
                                                              double amp, double2* __restrict__ out,
                                                              int* flag) {
  __shared__ double sx[kSrcChunk], sy[kSrcChunk], sz[kSrcChunk];
  __shared__ double2 tab[kPhaseN];
  fill_phase_table(tab);  // visible after the first barrier of the source loop
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = idx < n_pts;
  double x = 0, y = 0, z = 0;
  if (active) {
    x = pts[3 * idx];
    y = pts[3 * idx + 1];
    z = pts[3 * idx + 2];
  }
  double2 acc = make_double2(0.0, 0.0);
  bool bad = false;
  for (int base = 0; base < n_src; base += kSrcChunk) {
    __syncthreads();
    stage_sources(src, n_src, base, sx, sy, sz);
    __syncthreads();
    if (active) {
      const int n = min(kSrcChunk, n_src - base);
      #pragma unroll 4
      for (int j = 0; j < n; ++j) monopole_term<ATT>(x, y, z, sx[j], sy[j], sz[j], k1, kim, tab, acc, bad);
    }
  }
  if (active) {
    if (bad) atomicExch(flag, 1);
    out[idx] = make_double2(amp * acc.x, amp * acc.y);
  }
}

// Disc nodes of radiated_power: node (j, m) at (x_disc, r cos th, r sin th).
template <int ATT>
__global__ void __launch_bounds__(256) power_nodes_kernel(const double* __restrict__ src, int n_src,
                                                          double x_disc, double dr, double dth,
                                                          int n_r, int n_theta, double k1,
                                                          double kim, double amp,
                                                          double* __restrict__ node_out, int* flag) {
  __shared__ double sx[kSrcChunk], sy[kSrcChunk], sz[kSrcChunk];
  __shared__ double2 tab[kPhaseN];
  fill_phase_table(tab);  // visible after the first barrier of the source loop
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = idx < int64_t(n_r) * n_theta;
  double y = 0, z = 0;
  if (active) {
    const int j = int(idx / n_theta), m = int(idx % n_theta);
    const double r = (j + 0.5) * dr;
    const double th = (m + 0.5) * dth;
    y = r * cos(th);
    z = r * sin(th);
  }
  double2 acc = make_double2(0.0, 0.0);
  bool bad = false;
  for (int base = 0; base < n_src; base += kSrcChunk) {
    __syncthreads();
    stage_sources(src, n_src, base, sx, sy, sz);
    __syncthreads();
    if (active) {
      const int n = min(kSrcChunk, n_src - base);
      #pragma unroll 4
      for (int j = 0; j < n; ++j) monopole_term<ATT>(x_disc, y, z, sx[j], sy[j], sz[j], k1, kim, tab, acc, bad);
    }
  }
  if (active) {
    if (bad) atomicExch(flag, 1);
    const double re = amp * acc.x, im = amp * acc.y;
    node_out[idx] = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
  }
}

// ---------------------------------------------------------------------------- potential at points
// evaluate_potential_at (src/potential.cpp:161-201): u(x_m) = sum over voxels j with f_j != 0 of
// vol G(|x_m - c_j|) f_j, or self_weight(k, dx) f_j when |x_m - c_j| < 1e-9 dx.  O(N M) FP64: the
// Rayleigh term (phase table, refined rsqrt) times a complex weight.  Grid: point blocks x voxel
// chunk groups; a CTA stages kPotChunk consecutive voxels (whole or partial x-rows) in shared
// memory, vs threads share a point and split the chunk (vs: a power of two, larger for few
// points, so small point sets still fill the CTA), and each chunk group writes one
// partial sum per point; potential_reduce_kernel adds the groups in order (deterministic).
constexpr int kPotThreads = 256, kPotChunk = 768;  // 12 KB staged + 32 KB phase table + 4 KB: static smem

__global__ void phase_table_kernel(double2* tab) { fill_phase_table(tab); }

template <int ATT>
__global__ void __launch_bounds__(kPotThreads) potential_at_kernel(
    GridDev g, const double2* __restrict__ f, const double* __restrict__ pts, int64_t n_pts, double k1,
    double kim, double vol, double2 self, double coinc2, const double2* __restrict__ gtab,
    double2* __restrict__ partial, int vs) {
  __shared__ double2 fs[kPotChunk];  // vol * f of the staged voxels (self term: f, scaled back)
  __shared__ double2 tab[kPhaseN];
  __shared__ double2 red[kPotThreads];
  for (int j = threadIdx.x; j < kPhaseN; j += kPotThreads) tab[j] = gtab[j];
  const int pl = threadIdx.x / vs, sl = threadIdx.x % vs;
  const int64_t pt = int64_t(blockIdx.x) * (kPotThreads / vs) + pl;
  const bool active = pt < n_pts;
  double x0 = 0, x1 = 0, x2 = 0;
  if (active) {
    x0 = pts[3 * pt];
    x1 = pts[3 * pt + 1];
    x2 = pts[3 * pt + 2];
  }
  const int Nx = g.dims[0], Ny = g.dims[1];
  const int64_t count = int64_t(Nx) * Ny * g.dims[2];
  const int64_t nchunks = (count + kPotChunk - 1) / kPotChunk;
  const double inv_vol = 1.0 / vol;
  double2 a4[4];
  for (int c = 0; c < 4; ++c) a4[c] = make_double2(0.0, 0.0);
  bool bad = false;
  for (int64_t c = blockIdx.y; c < nchunks; c += gridDim.y) {
    const int64_t v0 = c * kPotChunk, v1 = min(count, v0 + kPotChunk);
    __syncthreads();  // previous chunk consumed (and, first time, the table staged)
    for (int64_t v = v0 + threadIdx.x; v < v1; v += kPotThreads) {
      const double2 x = f[v];
      fs[v - v0] = make_double2(vol * x.x, vol * x.y);
    }
    __syncthreads();
    if (!active) continue;
    for (int64_t gi = v0; gi < v1;) {  // row segments of the chunk
      const int64_t row = gi / Nx;
      const int jx0 = int(gi - row * Nx);
      const int64_t seg_end = min(v1, (row + 1) * Nx);
      const double cy = centre(g.lo[1], int(row % Ny), g.dx) - x1;  // src/potential.cpp:181-183
      const double cz = centre(g.lo[2], int(row / Ny), g.dx) - x2;
      const double ryz2 = fma(cz, cz, cy * cy);
      // branch-free term: a zero f_j adds an exact zero (the reference skips it, :186); a
      // coincident voxel (r < 1e-9 dx, :189-190) takes the self weight instead of G
      auto term = [&](int64_t q, double2& a) {
        const double2 fj = fs[q - v0];  // vol * f_j
        const double cx = centre(g.lo[0], jx0 + int(q - gi), g.dx) - x0;
        const double d2 = fma(cx, cx, ryz2);
        const bool co = d2 < coinc2;
        double2 gk = make_double2(0.0, 0.0);
        monopole_term_d2<ATT>(co ? 1.0 : d2, k1, kim, tab, gk, bad);  // e^{-Im k r} e^{i Re k r} / (4 pi r)
        const double wx = co ? self.x * inv_vol : gk.x, wy = co ? self.y * inv_vol : gk.y;
        a.x = fma(wx, fj.x, fma(-wy, fj.y, a.x));
        a.y = fma(wx, fj.y, fma(wy, fj.x, a.y));
      };
      const int o = int(gi - v0);
      int64_t q = gi + ((sl - o) % vs + vs) % vs;
      for (; q + 3 * vs < seg_end; q += 4 * vs) {  // four independent chains
        term(q, a4[0]);
        term(q + vs, a4[1]);
        term(q + 2 * vs, a4[2]);
        term(q + 3 * vs, a4[3]);
      }
      for (; q < seg_end; q += vs) term(q, a4[0]);
      gi = seg_end;
    }
  }
  double2 acc = make_double2((a4[0].x + a4[1].x) + (a4[2].x + a4[3].x), (a4[0].y + a4[1].y) + (a4[2].y + a4[3].y));
  red[threadIdx.x] = acc;
  __syncthreads();
  if (active && sl == 0) {
    double2 t = red[threadIdx.x];
    for (int q = 1; q < vs; ++q) t = make_double2(t.x + red[threadIdx.x + q].x, t.y + red[threadIdx.x + q].y);
    partial[int64_t(blockIdx.y) * n_pts + pt] = t;
  }
}

__global__ void potential_reduce_kernel(const double2* __restrict__ partial, int groups, int64_t n_pts,
                                        double2* __restrict__ out) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n_pts; p += int64_t(gridDim.x) * blockDim.x) {
    double2 t = make_double2(0.0, 0.0);
    for (int y = 0; y < groups; ++y) {
      const double2 v = partial[int64_t(y) * n_pts + p];
      t = make_double2(t.x + v.x, t.y + v.y);
    }
    out[p] = t;
  }
}

// Fixed-order reduction: ring j sums its n_theta nodes in order, times r_j; then rings in
// order. One block; deterministic for any launch configuration.
__global__ void power_reduce_kernel(const double* __restrict__ nodes, int n_r, int n_theta,
                                    double dr, double* __restrict__ rings, double* out,
                                    double factor) {
  for (int j = threadIdx.x; j < n_r; j += blockDim.x) {
    double ring = 0.0;
    for (int m = 0; m < n_theta; ++m) ring = __dadd_rn(ring, nodes[int64_t(j) * n_theta + m]);
    rings[j] = __dmul_rn(ring, (j + 0.5) * dr);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = 0.0;
    for (int j = 0; j < n_r; ++j) total = __dadd_rn(total, rings[j]);
    *out = total * factor;
  }
}

// rhs_source: out = coeff * sum_{m=1}^{n-1} p_m p_{n-m}, complex products as (ac-bd, ad+bc)
struct LowerPtrs {
  const double2* p[32];
};

__global__ void rhs_kernel(LowerPtrs lp, int n, int64_t count, double coeff,
                           double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int m = 1; m <= n - 1; ++m) {
      const double2 a = lp.p[m - 1][i], b = lp.p[n - m - 1][i];
      const double pr = __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
      const double pi = __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x));
      re = __dadd_rn(re, pr);
      im = __dadd_rn(im, pi);
    }
    out[i] = make_double2(__dmul_rn(coeff, re), __dmul_rn(coeff, im));
  }
}

// The full quadratic source of the paper's Eq. (cascade_1), truncated at the
// M harmonics held: sum_{m=1}^{n-1} p_m p_{n-m} + 2 sum_{m=n+1}^{M} p_m conj(p_{m-n}). The first
// sum is accumulated exactly as rhs_kernel (so M = n - 1 is bitwise fusg_rhs_source); the
// conjugate terms follow in increasing m. Used by iterated (Gauss-Seidel) sweeps, where the
// higher harmonics of the previous sweep are available.
__global__ void rhs_full_kernel(LowerPtrs lp, int n, int M, int64_t count, double coeff,
                                double2* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int m = 1; m <= n - 1; ++m) {
      const double2 a = lp.p[m - 1][i], b = lp.p[n - m - 1][i];
      re = __dadd_rn(re, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
      im = __dadd_rn(im, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    for (int m = n + 1; m <= M; ++m) {  // a * conj(b) = (ac + bd, bc - ad) with b = (c, d)
      const double2 a = lp.p[m - 1][i], b = lp.p[m - n - 1][i];
      const double pr = __dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
      const double pi = __dsub_rn(__dmul_rn(a.y, b.x), __dmul_rn(a.x, b.y));
      re = __dadd_rn(re, __dmul_rn(2.0, pr));
      im = __dadd_rn(im, __dmul_rn(2.0, pi));
    }
    out[i] = make_double2(__dmul_rn(coeff, re), __dmul_rn(coeff, im));
  }
}

// interpolate (src/grid.cpp:141-195), exact rounding
// Source cell and weight of target index i on axis a (src/grid.cpp:156-170): q = (p - lo_s)/dx_s
// - 0.5, base = clamp(floor q, 0, max(0, n - 2)), t = clamp(q - base, 0, 1) (t > 1 -> 1, or 0
// when n == 1); the same correctly rounded operations as the reference's non-FMA build.
__device__ __forceinline__ void interp_axis(const GridDev& s, const GridDev& t, int a, int i, int& base,
                                            double& frac) {
  const double p = centre(t.lo[a], i, t.dx);
  const double q = __dsub_rn(__ddiv_rn(__dsub_rn(p, s.lo[a]), s.dx), 0.5);
  int b = int(floor(q));
  const int hi = max(0, s.dims[a] - 2);
  b = b < 0 ? 0 : (b > hi ? hi : b);
  double fr = __dsub_rn(q, double(b));
  if (fr < 0.0) fr = 0.0;
  if (fr > 1.0) fr = s.dims[a] > 1 ? 1.0 : 0.0;
  base = b;
  frac = fr;
}

// Per-axis cells and weights (they depend on one index each), computed once per call.
// (t.dims[2] is the number of target planes computed, starting at target plane t.z_off.)
__global__ void interp_axes_kernel(GridDev s, GridDev t, int* __restrict__ base, double* __restrict__ frac) {
  const int n = t.dims[0] + t.dims[1] + t.dims[2];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int a = j < t.dims[0] ? 0 : (j < t.dims[0] + t.dims[1] ? 1 : 2);
    const int i = a == 0 ? j : (a == 1 ? j - t.dims[0] : j - t.dims[0] - t.dims[1] + t.z_off);
    interp_axis(s, t, a, i, base[j], frac[j]);
  }
}

// Trilinear gather (src/grid.cpp:171-192) from the per-axis tables: 32-bit index arithmetic,
// no divisions per point; consecutive threads take consecutive x.
__global__ void __launch_bounds__(256) interp_kernel(GridDev s, const double2* __restrict__ f, GridDev t,
                                                     const int* __restrict__ base, const double* __restrict__ frac,
                                                     double2* __restrict__ out) {
  const unsigned nx = unsigned(t.dims[0]), ny = unsigned(t.dims[1]);
  const unsigned count = nx * ny * unsigned(t.dims[2]);
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count; idx += gridDim.x * blockDim.x) {
    const unsigned r = idx / nx, ix = idx - r * nx;
    const unsigned iz = r / ny, iy = r - iz * ny;
    const int i0[3] = {__ldg(base + ix), __ldg(base + nx + iy), __ldg(base + nx + ny + iz)};
    const double tt[3] = {__ldg(frac + ix), __ldg(frac + nx + iy), __ldg(frac + nx + ny + iz)};
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int cz = 0; cz < 2; ++cz)
#pragma unroll
      for (int cy = 0; cy < 2; ++cy)
#pragma unroll
        for (int cx = 0; cx < 2; ++cx) {
          const double wx = cx ? tt[0] : __dsub_rn(1.0, tt[0]);
          const double wy = cy ? tt[1] : __dsub_rn(1.0, tt[1]);
          const double wz = cz ? tt[2] : __dsub_rn(1.0, tt[2]);
          const double wgt = __dmul_rn(__dmul_rn(wx, wy), wz);
          if (wgt == 0.0) continue;
          const int jx = min(max(i0[0] + cx, 0), s.dims[0] - 1);
          const int jy = min(max(i0[1] + cy, 0), s.dims[1] - 1);
          const int jz = min(max(i0[2] + cz, 0), s.dims[2] - 1);
          const double2 v = __ldg(f + jx + int64_t(s.dims[0]) * (jy + int64_t(s.dims[1]) * (jz - s.z_off)));
          re = __dadd_rn(re, __dmul_rn(wgt, v.x));
          im = __dadd_rn(im, __dmul_rn(wgt, v.y));
        }
    out[idx] = make_double2(re, im);
  }
}

// max |v| (for the 15 MPa weak-nonlinearity warning, src/cascade.cpp:56-60)
__global__ void max_abs_kernel(const double2* __restrict__ v, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, hypot(v[i].x, v[i].y));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// shrink_domain_by_threshold (src/grid.cpp:114-139): index bounding box of |f| >= threshold;
// block min/max reduction then one atomic per block (order independent: exact)
__global__ void threshold_box_kernel(GridDev g, const double2* __restrict__ f, double thr, int* __restrict__ box) {
  __shared__ int red[6][256];
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {-1, -1, -1};
  const int64_t count = int64_t(g.dims[0]) * g.dims[1] * g.dims[2];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    if (hypot(f[i].x, f[i].y) >= thr) {
      const int ix = int(i % g.dims[0]);
      const int64_t r = i / g.dims[0];
      const int ii[3] = {ix, int(r % g.dims[1]), int(r / g.dims[1])};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = min(lo[a], ii[a]);
        hi[a] = max(hi[a], ii[a]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    red[a][threadIdx.x] = lo[a];
    red[3 + a][threadIdx.x] = hi[a];
  }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        red[a][threadIdx.x] = min(red[a][threadIdx.x], red[a][threadIdx.x + w]);
        red[3 + a][threadIdx.x] = max(red[3 + a][threadIdx.x], red[3 + a][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&box[a], red[a][0]);
      atomicMax(&box[3 + a], red[3 + a][0]);
    }
}

// localisedness_map (src/analysis.cpp:80-90): log10(|f| / max|f|), -inf for zero voxels
__global__ void localisedness_kernel(const double2* __restrict__ f, int64_t n, double max_abs, double* __restrict__ q) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double a = hypot(f[i].x, f[i].y);
    q[i] = a > 0.0 ? log10(a / max_abs) : -CUDART_INF;
  }
}

// ---------------------------------------------------------------------------- launchers
// Attenuation mode for a launch: 0 if Im k == 0; 1 if Im k * dmax <= kPolyAttMax (dmax bounds
// every source-target distance); else 2.
static int att_mode(double kim, double dmax) {
  if (kim == 0.0) return 0;
  return (dmax >= 0.0 && kim * dmax <= kPolyAttMax) ? 1 : 2;
}

// Diagonal of the bounding box of the source points and a target box: bounds all distances.
double distance_bound(const double* src_host, int n_src, const double lo[3], const double hi[3]) {
  double blo[3] = {lo[0], lo[1], lo[2]}, bhi[3] = {hi[0], hi[1], hi[2]};
  for (int i = 0; i < n_src; ++i)
    for (int a = 0; a < 3; ++a) {
      blo[a] = std::min(blo[a], src_host[3 * i + a]);
      bhi[a] = std::max(bhi[a], src_host[3 * i + a]);
    }
  double d2 = 0.0;
  for (int a = 0; a < 3; ++a) d2 += (bhi[a] - blo[a]) * (bhi[a] - blo[a]);
  return std::sqrt(d2) * (1.0 + 1e-12);
}

#define FUSG_ATT_DISPATCH(att, KERNEL, ...)        \
  do {                                             \
    if ((att) == 0) KERNEL<0><<<__VA_ARGS__;       \
    else if ((att) == 1) KERNEL<1><<<__VA_ARGS__;  \
    else KERNEL<2><<<__VA_ARGS__;                  \
  } while (0)
static int grid_stride_blocks(const fusg_ctx* ctx, int64_t n, int threads) {
  const int64_t need = (n + threads - 1) / threads;
  const int64_t cap = int64_t(ctx->num_sms) * 16;
  return int(std::max<int64_t>(1, std::min(need, cap)));
}

fusg_status upload_sources(const double* src_host, int n_src, double** dev, cudaStream_t s) {
  if (n_src < 1) return set_error(FUSG_INVALID_ARGUMENT, "monopole sum: no source points");
  FUSG_CUDA_TRY(cudaMallocAsync(dev, sizeof(double) * 3 * n_src, s));
  FUSG_CUDA_TRY(cudaMemcpyAsync(*dev, src_host, sizeof(double) * 3 * n_src,
                                cudaMemcpyHostToDevice, s));
  return FUSG_OK;
}

static fusg_status check_flag(fusg_ctx* ctx, cudaStream_t s) {
  int h = 0;
  FUSG_CUDA_TRY(cudaMemcpyAsync(&h, ctx->dev_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  if (h) {
    FUSG_CUDA_TRY(cudaMemsetAsync(ctx->dev_flag, 0, sizeof(int), s));
    return set_error(FUSG_INVALID_ARGUMENT, "evaluation point coincides with a monopole source");
  }
  return FUSG_OK;
}

fusg_status monopole_grid(fusg_ctx* ctx, const double* src_dev, int n_src, const fusg_grid& g,
                          double kre, double kim, double amp, double2* out, cudaStream_t s,
                          double dmax, int z0, int nz) {
  GridDev gd = to_dev(g);
  if (nz >= 0) {  // z-slab [z0, z0 + nz) of g (p1 shards by z-planes)
    gd.dims[2] = nz;
    gd.z_off = z0;
  }
  const int64_t count = int64_t((gd.dims[0] + kVPT - 1) / kVPT) * gd.dims[1] * gd.dims[2];
  if (count == 0) return FUSG_OK;
  const int threads = FUSG_MONO_THREADS;
  const unsigned blocks = unsigned((count + threads - 1) / threads);
  const double k1 = phase_scale(kre, kGridPhaseBits);
  if (!(k1 > 0.0))  // the grid kernel measures distances in phase-table turns (Re k > 0)
    return set_error(FUSG_INVALID_ARGUMENT, "monopole_grid: Re k must be positive");
  // attenuating media: tabulated attenuation (ATT 3) when every Re k d / (2 pi) N fits the
  // coarse table (FUSG_ATT_TABLE=0 keeps the polynomial / exp() modes)
  static const bool att_table = [] {
    const char* e = getenv("FUSG_ATT_TABLE");
    return !(e && atoi(e) == 0);
  }();
  const double umax = dmax * k1;
  const int n_eh = dmax >= 0.0 ? int(umax / (1 << kGridPhaseBits)) + 2 : kEhMax + 1;
  const size_t dsm = sizeof(double2) * (size_t(kGridRep) << kGridPhaseBits) + sizeof(double) * kEhMax;
  static std::atomic<uint64_t> attr_mask{0};
  const bool attr = once_per_device(attr_mask, [&] {
    for (auto fn : {monopole_grid_kernel<0>, monopole_grid_kernel<1>, monopole_grid_kernel<2>, monopole_grid_kernel<3>})
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dsm)) != cudaSuccess) return false;
    return true;
  });
  if (!attr) return set_error(FUSG_CUDA, "monopole_grid: cannot configure shared memory");
  if (att_table && kim > 0.0 && k1 > 0.0 && n_eh <= kEhMax && umax < 1e9) {
    monopole_grid_kernel<3><<<blocks, threads, dsm, s>>>(src_dev, n_src, gd, k1, kim / k1, amp, out,
                                                         ctx->dev_flag, n_eh);
  } else {
    FUSG_ATT_DISPATCH(att_mode(kim, dmax), monopole_grid_kernel, blocks, threads, dsm, s>>>(
                          src_dev, n_src, gd, k1, kim / k1, amp, out, ctx->dev_flag));
  }
  ctx->launches++;
  FUSG_LAUNCH_CHECK("monopole_grid_kernel");
  return FUSG_OK;
}

// Host restatement of interp_axis's z cell (same IEEE operations, no contraction): the source
// planes [lo, hi] the target planes [tz0, tz0 + tnz) read (the z-slab transfer's halo).
static void interp_source_planes(const fusg_grid& src, const fusg_grid& tgt, int tz0, int tnz, int* lo, int* hi) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int iz = tz0; iz < tz0 + tnz; ++iz) {
    const double p = tgt.lo[2] + (double(iz) + 0.5) * tgt.dx;
    const double q = (p - src.lo[2]) / src.dx - 0.5;
    int b = int(std::floor(q));
    const int top = std::max(0, src.dims[2] - 2);
    b = b < 0 ? 0 : (b > top ? top : b);
    mn = std::min(mn, b);
    mx = std::max(mx, std::min(b + 1, src.dims[2] - 1));
  }
  *lo = mn;
  *hi = mx;
}

// Target planes [tz0, tz0 + tnz) from source planes [sz0, sz0 + snz) held in f (a z-slab of the
// source field, halo included); the full transfer is tz0 = sz0 = 0, tnz = tgt dims, snz = src dims.
static fusg_status interpolate_slab_dev(fusg_ctx* ctx, const fusg_grid& src, int sz0, int snz, const double2* f,
                                        const fusg_grid& tgt, int tz0, int tnz, double2* out, cudaStream_t s) {
  for (int a = 0; a < 3; ++a)
    if (tgt.lo[a] < src.lo[a] - src.dx || tgt.hi[a] > src.hi[a] + src.dx)
      return set_error(FUSG_INVALID_ARGUMENT,
                       "interpolate: target extends more than one source voxel beyond the source domain");
  if (tz0 < 0 || tnz < 0 || int64_t(tz0) + tnz > tgt.dims[2] || sz0 < 0 || snz < 0 ||
      int64_t(sz0) + snz > src.dims[2])
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate: slab outside the grid");
  if (tnz == 0) return FUSG_OK;
  int need_lo, need_hi;
  interp_source_planes(src, tgt, tz0, tnz, &need_lo, &need_hi);
  if (need_lo < sz0 || need_hi >= sz0 + snz)
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate: the source slab lacks planes " + std::to_string(need_lo) +
                                                ".." + std::to_string(need_hi) + " the target slab reads");
  const int64_t count = int64_t(tgt.dims[0]) * tgt.dims[1] * tnz;
  if (count >= (int64_t(1) << 32))
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate: target above 2^32 voxels");
  GridDev sd = to_dev(src), td = to_dev(tgt);
  sd.z_off = sz0;
  td.dims[2] = tnz;
  td.z_off = tz0;
  const int nax = tgt.dims[0] + tgt.dims[1] + tnz;
  void* tabs = nullptr;
  FUSG_CUDA_TRY(cudaMallocAsync(&tabs, size_t(nax) * (sizeof(int) + sizeof(double)) + 16, s));
  double* frac = static_cast<double*>(tabs);
  int* base = reinterpret_cast<int*>(frac + nax);
  interp_axes_kernel<<<(nax + 255) / 256, 256, 0, s>>>(sd, td, base, frac);
  interp_kernel<<<grid_stride_blocks(ctx, count, 256), 256, 0, s>>>(sd, f, td, base, frac, out);
  ctx->launches += 2;
  FUSG_CUDA_TRY(cudaFreeAsync(tabs, s));
  FUSG_LAUNCH_CHECK("interp_kernel");
  return FUSG_OK;
}

fusg_status interpolate_dev(fusg_ctx* ctx, const fusg_grid& src, const double2* f,
                            const fusg_grid& tgt, double2* out, cudaStream_t s) {
  return interpolate_slab_dev(ctx, src, 0, src.dims[2], f, tgt, 0, tgt.dims[2], out, s);
}

fusg_status rhs_dev(fusg_ctx* ctx, int n, const double2* const* lower, int64_t count, double coeff,
                    double2* out, cudaStream_t s) {
  if (n < 2) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source: harmonic index must be >= 2");
  if (n - 1 > 32) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source: at most 33 harmonics");
  LowerPtrs lp{};
  for (int m = 0; m < n - 1; ++m) {
    if (!lower[m]) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source: null lower harmonic");
    lp.p[m] = lower[m];
  }
  rhs_kernel<<<grid_stride_blocks(ctx, count, 256), 256, 0, s>>>(lp, n, count, coeff, out);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("rhs_kernel");
  return FUSG_OK;
}

fusg_status rhs_full_dev(fusg_ctx* ctx, int n, const double2* const* fields, int M, int64_t count,
                         double coeff, double2* out, cudaStream_t s) {
  if (n < 2) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source: harmonic index must be >= 2");
  if (M < n - 1) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source_full: need p_1 .. p_{n-1}");
  if (M > 32) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source_full: at most 32 harmonics");
  LowerPtrs lp{};
  for (int m = 0; m < M; ++m) {  // p_n enters through p_{2n} conj(p_n) when 2n <= M
    if (!fields[m] && m != n - 1) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source_full: null harmonic field");
    if (!fields[m] && 2 * n <= M) return set_error(FUSG_INVALID_ARGUMENT, "rhs_source_full: p_n is needed when 2n <= M");
    lp.p[m] = fields[m];
  }
  rhs_full_kernel<<<grid_stride_blocks(ctx, count, 256), 256, 0, s>>>(lp, n, M, count, coeff, out);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("rhs_full_kernel");
  return FUSG_OK;
}

fusg_status max_abs_dev(fusg_ctx* ctx, const double2* v, int64_t n, double* out, cudaStream_t s) {
  unsigned long long* d = nullptr;
  FUSG_CUDA_TRY(cudaMallocAsync(&d, sizeof(unsigned long long), s));
  FUSG_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
  max_abs_kernel<<<grid_stride_blocks(ctx, n, 256), 256, 0, s>>>(v, n, d);
  ctx->launches++;
  unsigned long long h = 0;
  FUSG_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  FUSG_CUDA_TRY(cudaFreeAsync(d, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  double m;
  memcpy(&m, &h, sizeof(m));
  *out = m;
  return FUSG_OK;
}

fusg_status radiated_power_dev(fusg_ctx* ctx, const double* src_dev, int n_src, double x_disc,
                               double R, double kre, double kim, double amp, double rho0, double c0,
                               int n_r, int n_theta, double* out_host, cudaStream_t s, double dmax) {
  if (n_r < 1 || n_theta < 1) return set_error(FUSG_INVALID_ARGUMENT, "radiated_power: empty disc");
  const double dr = R / n_r;
  const double dth = 2.0 * M_PI / n_theta;
  const int64_t nn = int64_t(n_r) * n_theta;
  double* nodes = nullptr;
  FUSG_CUDA_TRY(cudaMallocAsync(&nodes, sizeof(double) * (nn + n_r + 1), s));
  FUSG_ATT_DISPATCH(att_mode(kim, dmax), power_nodes_kernel, unsigned((nn + 255) / 256), 256, 0, s>>>(
                        src_dev, n_src, x_disc, dr, dth, n_r, n_theta, phase_scale(kre), kim, amp, nodes,
                        ctx->dev_flag));
  ctx->launches++;
  FUSG_LAUNCH_CHECK("power_nodes_kernel");
  // the final total * dr * dth / (2 rho0 c0) is applied on the host in the reference's order
  power_reduce_kernel<<<1, 256, 0, s>>>(nodes, n_r, n_theta, dr, nodes + nn, nodes + nn + n_r, 1.0);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("power_reduce_kernel");
  double total = 0.0;
  FUSG_CUDA_TRY(cudaMemcpyAsync(&total, nodes + nn + n_r, sizeof(double), cudaMemcpyDeviceToHost, s));
  FUSG_CUDA_TRY(cudaFreeAsync(nodes, s));
  fusg_status st = check_flag(ctx, s);
  if (st != FUSG_OK) return st;
  *out_host = total * dr * dth / (2.0 * rho0 * c0);
  return FUSG_OK;
}

fusg_status check_monopole_flag(fusg_ctx* ctx, cudaStream_t s) { return check_flag(ctx, s); }

}  // namespace fusg

using namespace fusg;

extern "C" {

fusg_status fusg_monopole_grid(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                               const fusg_grid* grid, double k_re, double k_im, double amp,
                               double* out_dev, void* stream) {
  if (!ctx || !grid || !out_dev) return set_error(FUSG_INVALID_ARGUMENT, "monopole_grid: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->pick(stream);
  double* src = nullptr;
  fusg_status st = upload_sources(src_host, n_src, &src, s);
  if (st != FUSG_OK) return st;
  st = monopole_grid(ctx, src, n_src, *grid, k_re, k_im, amp, reinterpret_cast<double2*>(out_dev), s,
                     distance_bound(src_host, n_src, grid->lo, grid->hi));
  cudaFreeAsync(src, s);
  if (st != FUSG_OK) return st;
  return check_flag(ctx, s);
}

fusg_status fusg_monopole_grid_zslab(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                                     const fusg_grid* grid, int32_t z0, int32_t nz, double k_re,
                                     double k_im, double amp, double* out_dev, void* stream) {
  if (!ctx || !grid || (nz > 0 && !out_dev))
    return set_error(FUSG_INVALID_ARGUMENT, "monopole_grid_zslab: null argument");
  if (z0 < 0 || nz < 0 || int64_t(z0) + nz > grid->dims[2])
    return set_error(FUSG_INVALID_ARGUMENT, "monopole_grid_zslab: slab outside the grid");
  if (nz == 0) return FUSG_OK;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->pick(stream);
  double* src = nullptr;
  fusg_status st = upload_sources(src_host, n_src, &src, s);
  if (st != FUSG_OK) return st;
  st = monopole_grid(ctx, src, n_src, *grid, k_re, k_im, amp, reinterpret_cast<double2*>(out_dev), s,
                     distance_bound(src_host, n_src, grid->lo, grid->hi), z0, nz);
  cudaFreeAsync(src, s);
  if (st != FUSG_OK) return st;
  return check_flag(ctx, s);
}

fusg_status fusg_monopole_points(fusg_ctx* ctx, const double* src_host, int32_t n_src,
                                 const double* pts_dev, int64_t n_pts, double k_re, double k_im,
                                 double amp, double* out_dev, void* stream) {
  if (!ctx || (n_pts > 0 && (!pts_dev || !out_dev)))
    return set_error(FUSG_INVALID_ARGUMENT, "monopole_points: null argument");
  if (n_pts == 0) return FUSG_OK;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->pick(stream);
  double* src = nullptr;
  fusg_status st = upload_sources(src_host, n_src, &src, s);
  if (st != FUSG_OK) return st;
  FUSG_ATT_DISPATCH(att_mode(k_im, -1.0), monopole_points_kernel, unsigned((n_pts + 255) / 256), 256,
                    0, s>>>(src, n_src, pts_dev, n_pts, phase_scale(k_re), k_im, amp,
                            reinterpret_cast<double2*>(out_dev), ctx->dev_flag));
  ctx->launches++;
  FUSG_LAUNCH_CHECK("monopole_points_kernel");
  cudaFreeAsync(src, s);
  return check_flag(ctx, s);
}

// evaluate_potential_at (src/potential.cpp:161-201)
fusg_status fusg_evaluate_potential_at(fusg_ctx* ctx, const fusg_grid* grid, const fusg_wavenumber* k,
                                       const double* f_dev, const double* pts_host, int64_t n_pts,
                                       double* out_host) {
  if (!ctx || !grid || !k || (n_pts > 0 && (!f_dev || !pts_host || !out_host)))
    return set_error(FUSG_INVALID_ARGUMENT, "evaluate_potential_at: null argument");
  if (n_pts < 0) return set_error(FUSG_INVALID_ARGUMENT, "evaluate_potential_at: negative point count");
  if (n_pts == 0) return FUSG_OK;
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  if (!ctx->phase_tab) {
    FUSG_CUDA_TRY(cudaMalloc(&ctx->phase_tab, sizeof(double2) * kPhaseN));
    phase_table_kernel<<<1, 256, 0, s>>>(ctx->phase_tab);
    ctx->launches++;
    FUSG_LAUNCH_CHECK("phase_table_kernel");
  }
  double sw[2];
  FUSG_TRY(fusg_self_weight(k, grid->dx, sw));
  const GridDev g = to_dev(*grid);
  const int64_t count = int64_t(g.dims[0]) * g.dims[1] * g.dims[2];
  const int64_t nchunks = (count + kPotChunk - 1) / kPotChunk;
  // threads per point: 4 for large point sets, up to the whole CTA for a handful of points
  int vs = 4;
  while (vs < kPotThreads && int64_t(kPotThreads / vs) > n_pts * 2) vs *= 2;
  const int pb = kPotThreads / vs;
  const int64_t pblocks = (n_pts + pb - 1) / pb;
  // one full wave of resident CTAs (chunk groups loop over their chunks); one partial per
  // (chunk group, point)
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, potential_at_kernel<2>, kPotThreads, 0);
  per_sm = std::max(per_sm, 1);
  const int64_t wave = int64_t(ctx->num_sms) * per_sm;
  const int groups = int(std::max<int64_t>(1, std::min<int64_t>(nchunks, std::max<int64_t>(1, wave / pblocks))));
  double *pts = nullptr;
  double2 *partial = nullptr, *out = nullptr;
  FUSG_CUDA_TRY(cudaMallocAsync(&pts, sizeof(double) * 3 * n_pts, s));
  FUSG_CUDA_TRY(cudaMallocAsync(&partial, sizeof(double2) * n_pts * groups, s));
  FUSG_CUDA_TRY(cudaMallocAsync(&out, sizeof(double2) * n_pts, s));
  FUSG_CUDA_TRY(cudaMemcpyAsync(pts, pts_host, sizeof(double) * 3 * n_pts, cudaMemcpyHostToDevice, s));
  // distance bound: grid box vs the points' bounding box (attenuation polynomial eligibility)
  double blo[3] = {grid->lo[0], grid->lo[1], grid->lo[2]}, bhi[3] = {grid->hi[0], grid->hi[1], grid->hi[2]};
  for (int64_t i = 0; i < n_pts; ++i)
    for (int a = 0; a < 3; ++a) {
      blo[a] = std::min(blo[a], pts_host[3 * i + a]);
      bhi[a] = std::max(bhi[a], pts_host[3 * i + a]);
    }
  double dd = 0.0;
  for (int a = 0; a < 3; ++a) dd += (bhi[a] - blo[a]) * (bhi[a] - blo[a]);
  const double coinc = 1e-9 * grid->dx;
  FUSG_ATT_DISPATCH(att_mode(k->k_im, std::sqrt(dd) * (1.0 + 1e-12)), potential_at_kernel,
                    dim3(unsigned(pblocks), unsigned(groups)), kPotThreads, 0,
                    s>>>(g, reinterpret_cast<const double2*>(f_dev), pts, n_pts, phase_scale(k->k_re), k->k_im,
                         grid->dx * grid->dx * grid->dx, make_double2(sw[0], sw[1]), coinc * coinc,
                         ctx->phase_tab, partial, vs));
  ctx->launches++;
  FUSG_LAUNCH_CHECK("potential_at_kernel");
  potential_reduce_kernel<<<grid_stride_blocks(ctx, n_pts, 256), 256, 0, s>>>(partial, groups, n_pts, out);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("potential_reduce_kernel");
  FUSG_CUDA_TRY(cudaMemcpyAsync(out_host, out, sizeof(double2) * n_pts, cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(pts, s);
  cudaFreeAsync(partial, s);
  cudaFreeAsync(out, s);
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

fusg_status fusg_field_threshold_box(fusg_ctx* ctx, const fusg_grid* grid, const double* f_dev, double q0,
                                     int32_t lo_idx[3], int32_t hi_idx[3], double* max_abs_out) {
  if (!ctx || !grid || !f_dev || !lo_idx || !hi_idx)
    return set_error(FUSG_INVALID_ARGUMENT, "threshold_box: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const GridDev g = to_dev(*grid);
  const int64_t count = int64_t(g.dims[0]) * g.dims[1] * g.dims[2];
  double m = 0.0;
  FUSG_TRY(max_abs_dev(ctx, reinterpret_cast<const double2*>(f_dev), count, &m, s));
  if (max_abs_out) *max_abs_out = m;
  if (m <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "shrink_domain_by_threshold: field is identically zero");
  const double thr = (q0 >= 0.0) ? m : m * std::pow(10.0, q0);  // q0 >= 0 keeps only the maximum
  int* box = nullptr;
  FUSG_CUDA_TRY(cudaMallocAsync(&box, 6 * sizeof(int), s));
  const int init[6] = {INT_MAX, INT_MAX, INT_MAX, -1, -1, -1};
  FUSG_CUDA_TRY(cudaMemcpyAsync(box, init, sizeof(init), cudaMemcpyHostToDevice, s));
  threshold_box_kernel<<<grid_stride_blocks(ctx, count, 256), 256, 0, s>>>(g, reinterpret_cast<const double2*>(f_dev),
                                                                            thr, box);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("threshold_box_kernel");
  int h[6];
  FUSG_CUDA_TRY(cudaMemcpyAsync(h, box, sizeof(h), cudaMemcpyDeviceToHost, s));
  FUSG_CUDA_TRY(cudaFreeAsync(box, s));
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  for (int a = 0; a < 3; ++a) {
    lo_idx[a] = h[a];
    hi_idx[a] = h[3 + a];
  }
  return FUSG_OK;
}

fusg_status fusg_localisedness_map(fusg_ctx* ctx, const double* f_dev, int64_t count, double* q_dev) {
  if (!ctx || (count > 0 && (!f_dev || !q_dev))) return set_error(FUSG_INVALID_ARGUMENT, "localisedness_map: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  double m = 0.0;
  FUSG_TRY(max_abs_dev(ctx, reinterpret_cast<const double2*>(f_dev), count, &m, s));
  if (m <= 0.0) return set_error(FUSG_INVALID_ARGUMENT, "localisedness_map: field is identically zero");
  localisedness_kernel<<<grid_stride_blocks(ctx, count, 256), 256, 0, s>>>(reinterpret_cast<const double2*>(f_dev),
                                                                           count, m, q_dev);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("localisedness_kernel");
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

fusg_status fusg_radiated_power(fusg_ctx* ctx, const double* src_host, int32_t n_src, double x_disc,
                                double R, double k_re, double k_im, double amp, double rho0,
                                double c0, int32_t n_r, int32_t n_theta, double* out_host) {
  if (!ctx || !out_host) return set_error(FUSG_INVALID_ARGUMENT, "radiated_power: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  double* src = nullptr;
  fusg_status st = upload_sources(src_host, n_src, &src, s);
  if (st != FUSG_OK) return st;
  const double dlo[3] = {x_disc, -R, -R}, dhi[3] = {x_disc, R, R};
  st = radiated_power_dev(ctx, src, n_src, x_disc, R, k_re, k_im, amp, rho0, c0, n_r, n_theta,
                          out_host, s, distance_bound(src_host, n_src, dlo, dhi));
  cudaFreeAsync(src, s);
  return st;
}

fusg_status fusg_rhs_source(fusg_ctx* ctx, int32_t n, const double* const* lower_dev, int64_t count,
                            const fusg_medium* m, double omega, double* out_dev, void* stream) {
  if (!ctx || !m || !lower_dev || !out_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "rhs_source: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  const double coeff = fusg_rhs_coefficient(m, omega, n);
  return rhs_dev(ctx, n, reinterpret_cast<const double2* const*>(lower_dev), count, coeff,
                 reinterpret_cast<double2*>(out_dev), ctx->pick(stream));
}

fusg_status fusg_rhs_source_full(fusg_ctx* ctx, int32_t n, const double* const* fields_dev, int32_t M,
                                 int64_t count, const fusg_medium* m, double omega, double* out_dev,
                                 void* stream) {
  if (!ctx || !m || !fields_dev || !out_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "rhs_source_full: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  const double coeff = fusg_rhs_coefficient(m, omega, n);
  return rhs_full_dev(ctx, n, reinterpret_cast<const double2* const*>(fields_dev), M, count, coeff,
                      reinterpret_cast<double2*>(out_dev), ctx->pick(stream));
}

fusg_status fusg_interpolate_source_planes(const fusg_grid* src, const fusg_grid* target, int32_t tz0,
                                           int32_t tnz, int32_t* z_lo, int32_t* z_hi) {
  if (!src || !target || !z_lo || !z_hi || tnz < 1 || tz0 < 0 || int64_t(tz0) + tnz > target->dims[2])
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate_source_planes: bad argument");
  int lo, hi;
  interp_source_planes(*src, *target, tz0, tnz, &lo, &hi);
  *z_lo = lo;
  *z_hi = hi;
  return FUSG_OK;
}

fusg_status fusg_interpolate_zslab(fusg_ctx* ctx, const fusg_grid* src, int32_t sz0, int32_t snz,
                                   const double* f_slab_dev, const fusg_grid* target, int32_t tz0, int32_t tnz,
                                   double* out_dev, void* stream) {
  if (!ctx || !src || !target || (tnz > 0 && (!f_slab_dev || !out_dev)))
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate_zslab: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  return interpolate_slab_dev(ctx, *src, sz0, snz, reinterpret_cast<const double2*>(f_slab_dev), *target, tz0, tnz,
                              reinterpret_cast<double2*>(out_dev), ctx->pick(stream));
}

fusg_status fusg_interpolate(fusg_ctx* ctx, const fusg_grid* src, const double* f_dev,
                             const fusg_grid* target, double* out_dev, void* stream) {
  if (!ctx || !src || !target || !f_dev || !out_dev)
    return set_error(FUSG_INVALID_ARGUMENT, "interpolate: null argument");
  FUSG_CUDA_TRY(cudaSetDevice(ctx->device));
  return interpolate_dev(ctx, *src, reinterpret_cast<const double2*>(f_dev), *target,
                         reinterpret_cast<double2*>(out_dev), ctx->pick(stream));
}

}  // extern "C"
