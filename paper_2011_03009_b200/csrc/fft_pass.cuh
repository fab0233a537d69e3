// Batched 1D Stockham FFT passes over one axis of a 3D complex128 box.
//
// One CTA transforms a tile of T lines that are adjacent in memory along the contiguous
// (x) direction, so every global access moves T*16 contiguous bytes per line position
// (T = 8 -> full 128-byte lines).  The tile is staged in shared memory as [position][T].
// Stage 1 reads global memory straight into registers (pruned: positions >= nvalid are
// zero and never loaded) and the last stage writes global memory straight from registers
// (pruned: only positions < nvalid are stored); the stages between exchange through
// shared memory.  Loader/storer functors give each pass its addressing and fusions
// (zero padding, kernel generation, octant folding, spectral multiply, crop and scale).
//
// Stockham autosort, radix R, Ns = product of the radices already applied:
//   j in [0, L/R): k = j mod Ns; v[r] = x[j + r L/R] * w_{Ns R}^{r k}; v = DFT_R(v);
//   y[(j / Ns) Ns R + k + r Ns] = v[r]
//
// Endpoints see (pos, e): pos is the line position, e in [0, kMaxElems) the thread-local
// element slot (compile-time after unrolling), so an endpoint may keep per-element state in
// registers (pass C's spectral multiply does).
#pragma once
#include <cstdint>

#include "dft.cuh"
#include "plan.hpp"

namespace fusg {

// Shared tile [pos][T] with an XOR swizzle inside each row: element (pos, t) lives in slot
// t ^ (pos mod T).  Column-side accesses (a warp = T lines x a few positions) stay permutations
// of whole rows, and line-major accesses (a warp = one line x 32 positions, used to stage rows
// coalesced) hit distinct banks.
template <int T>
__device__ __forceinline__ int tidx(int pos, int t) {
  return pos * T + (t ^ (pos & (T - 1)));
}

// ------------------------------------------------------------------ stage
// One Stockham stage of runtime radix R in {2,3,4,5,7,8}.  A thread owns up to
// B = kMaxElems / R butterflies (j = jt + b * tpl); their values live in one fixed register
// array v[kMaxElems] whose element e maps to (b, r) = (e / R, e % R).  Element indices are
// compile-time everywhere (unrolled loops, per-radix switch arms), so v stays in registers.
template <bool INV>
__device__ __forceinline__ void dft_block(int R, double2* v) {
  static_assert(kMaxElems == 8, "dft_block is written for 8 elements per thread");
  switch (R) {
    case 2:
#pragma unroll
      for (int b = 0; b < 4; ++b) dft<2, INV>(v + 2 * b);
      break;
    case 3:
#pragma unroll
      for (int b = 0; b < 2; ++b) dft<3, INV>(v + 3 * b);
      break;
    case 4:
#pragma unroll
      for (int b = 0; b < 2; ++b) dft<4, INV>(v + 4 * b);
      break;
    case 5: dft<5, INV>(v); break;
    case 7: dft<7, INV>(v); break;
    case 8: dft<8, INV>(v); break;
    default: break;
  }
}

// slot e -> (b, r) for radix R
__device__ __forceinline__ void slot(int e, int R, int& b, int& r) {
  b = e / R;
  r = e - b * R;
}

template <bool INV, int T, bool FIRST, bool LAST, class Src, class Dst>
__device__ __forceinline__ void fft_stage(const AxisPlan& pl, int R, int Ns, double2* sm, int t,
                                          int jt, Src& src, Dst& dst) {
  const int L = pl.L;
  const int nb = L / R;
  const int B = kMaxElems / R;
  const int tws = L / (Ns * R);
  double2 v[kMaxElems];
#pragma unroll
  for (int e = 0; e < kMaxElems; ++e) {
    int b, r;
    slot(e, R, b, r);
    const int j = jt + b * pl.tpl;
    v[e] = make_double2(0.0, 0.0);
    if (b < B && j < nb) {
      const int pos = j + r * nb;
      v[e] = FIRST ? src.load(pos, e) : sm[tidx<T>(pos, t)];
    }
  }
  // everyone has read this stage's shared-memory inputs before anyone overwrites them
  if ((!FIRST || Src::kSmem) && (!LAST || Dst::kSmem)) __syncthreads();
  if (Ns > 1) {
#pragma unroll
    for (int e = 0; e < kMaxElems; ++e) {
      int b, r;
      slot(e, R, b, r);
      const int j = jt + b * pl.tpl;
      if (r > 0 && b < B && j < nb) {
        const int k = j % Ns;
        const double2 w = __ldg(&pl.tw[r * k * tws]);
        v[e] = INV ? cmulc(v[e], w) : cmul(v[e], w);
      }
    }
  }
  dft_block<INV>(R, v);
#pragma unroll
  for (int e = 0; e < kMaxElems; ++e) {
    int b, r;
    slot(e, R, b, r);
    const int j = jt + b * pl.tpl;
    if (b < B && j < nb) {
      const int k = j % Ns;
      const int p = (j - k) * R + k + r * Ns;  // (j / Ns) * Ns * R + k + r Ns
      if (LAST) dst.store(p, e, v[e]);
      else sm[tidx<T>(p, t)] = v[e];
    }
  }
  if (!LAST) __syncthreads();  // outputs visible to the next stage (a smem-backed Dst syncs in the caller)
}

template <bool INV, int T, class Src, class Dst>
__device__ __forceinline__ void fft_line(const AxisPlan& pl, double2* sm, int t, int jt, Src& src,
                                         Dst& dst) {
  const int n = pl.nst;
  if (n == 1) {
    fft_stage<INV, T, true, true>(pl, pl.radix[0], 1, sm, t, jt, src, dst);
    return;
  }
  fft_stage<INV, T, true, false>(pl, pl.radix[0], 1, sm, t, jt, src, dst);
  for (int s = 1; s < n - 1; ++s)
    fft_stage<INV, T, false, false>(pl, pl.radix[s], pl.ns[s], sm, t, jt, src, dst);
  fft_stage<INV, T, false, true>(pl, pl.radix[n - 1], pl.ns[n - 1], sm, t, jt, src, dst);
}

// Position of element slot e in the first stage (its read position), or -1 if unused.
__device__ __forceinline__ int first_stage_pos(const AxisPlan& pl, int jt, int e) {
  const int R = pl.radix[0];
  const int nb = pl.L / R;
  int b, r;
  slot(e, R, b, r);
  const int j = jt + b * pl.tpl;
  return (b < kMaxElems / R && j < nb) ? j + r * nb : -1;
}

// ------------------------------------------------------------------ line addressing
// A pass transforms lines (i, k): i in [0, n_inner) is tiled T at a time, k in [0, n_outer).
struct LineGeom {
  int n_inner, n_outer, ntiles;
};

// Plain strided global load with zero padding beyond nvalid (pruned input).
struct GLoad {
  const double2* p;
  int64_t si, sk, sp;
  int nvalid;
};
struct GLoadAt {
  static constexpr bool kSmem = false;
  const double2* base;
  int64_t sp;
  int nvalid;
  bool ok;
  __device__ __forceinline__ double2 load(int pos, int) const {
    if (ok && pos < nvalid) return __ldg(base + pos * sp);
    return make_double2(0.0, 0.0);
  }
};

// Plain strided global store of positions < nvalid (pruned output), times scale.
// first > 0 (kernel-spectrum build of an x-slab kernel): only positions [first, nvalid) are
// stored, position pos at (pos - first) * sp.
struct GStore {
  double2* p;
  int64_t si, sk, sp;
  int nvalid;
  double scale;  // 1.0 -> no multiply
  int first = 0;
};
struct GStoreAt {
  static constexpr bool kSmem = false;
  double2* base;
  int64_t sp;
  int nvalid;
  bool ok;
  double scale;
  int first;
  __device__ __forceinline__ void store(int pos, int, double2 v) const {
    if (ok && pos >= first && pos < nvalid) base[(pos - first) * sp] = (scale == 1.0) ? v : cscale(v, scale);
  }
};

// Shared-memory endpoint (used between fused transforms).
template <int T>
struct SmemIO {
  static constexpr bool kSmem = true;
  double2* sm;
  int t;
  __device__ __forceinline__ double2 load(int pos, int) const { return sm[tidx<T>(pos, t)]; }
  __device__ __forceinline__ void store(int pos, int, double2 v) const { sm[tidx<T>(pos, t)] = v; }
};

// Register endpoint: the last stage of one transform hands its outputs to the first stage
// of the next in registers (valid when the first stage reads exactly the positions the last
// stage wrote, i.e. equal first/last radix).
struct RegIO {
  static constexpr bool kSmem = false;
  double2 v[kMaxElems];
  __device__ __forceinline__ void store(int, int e, double2 x) { v[e] = x; }
};

__host__ __device__ __forceinline__ int fold_index(int k, int P) { return (2 * k <= P) ? k : P - k; }

// Wrapped signed offset (src/potential.cpp:88-94); kExcluded marks the never-touched band.
constexpr int kExcluded = -2147483647 - 1;
__host__ __device__ __forceinline__ int offset_of(int m, int count, int padded) {
  if (m < count) return m;
  if (m > padded - count) return m - padded;
  return kExcluded;
}

}  // namespace fusg
