// Loaders/storers of the FFT passes and the compile-time-planned (static) CTA kernels with
// their dispatch-table entry type.  Shared by volume_potential.cu (hand-tuned entries, the
// runtime-planned and warp kernels) and the generated static_gen_*.cu translation units (a
// ladder of padded lengths, tools/gen_static.py), which compile in parallel.
#pragma once
#include <cstddef>
#include <cmath>
#include <type_traits>

#include "fft_warp.cuh"

namespace fusg {

// ---------------------------------------------------------------------------- loaders
struct GLoadF {
  GLoad g;
  __device__ __forceinline__ GLoadAt at(int i, int k, bool ok) const {
    return GLoadAt{g.p + i * g.si + k * g.sk, g.sp, g.nvalid, ok};
  }
};
struct GStoreF {
  GStore g;
  __device__ __forceinline__ GStoreAt at(int i, int k, bool ok) const {
    return GStoreAt{g.p + i * g.si + k * g.sk, g.sp, g.nvalid, ok, g.scale, g.first};
  }
};

// Kernel-tensor generator for the first build pass (src/potential.cpp:96-115): line i is
// the non-negative offset pair (oy, oz) = (i mod Ny, i / Ny); position = x index of the
// padded box.
struct KGenAt {
  static constexpr bool kSmem = false;
  int Nx, Px, oy, oz;
  double dx, vol, kre, kim;
  double2 self;
  bool ok;
  __device__ __forceinline__ double2 load(int pos, int) const {
    const int ox = offset_of(pos, Nx, Px);
    if (!ok || ox == kExcluded) return make_double2(0.0, 0.0);
    if (ox == 0 && oy == 0 && oz == 0) return self;
    const double r = dx * sqrt(double(ox) * ox + double(oy) * oy + double(oz) * oz);
    const double mag = exp(-kim * r) / (4.0 * M_PI * r);
    double s, c;
    sincos(kre * r, &s, &c);
    return make_double2(vol * (mag * c), vol * (mag * s));
  }
};
struct KGenF {
  int Nx, Ny, Px;
  double dx, vol, kre, kim;
  double2 self;
  __device__ __forceinline__ KGenAt at(int i, int, bool ok) const {
    return KGenAt{Nx, Px, i % Ny, i / Ny, dx, vol, kre, kim, self, ok};
  }
};

// Even extension of a half-range line: value at padded position = base[|offset|].
struct FoldAt {
  static constexpr bool kSmem = false;
  const double2* base;
  int64_t sp;
  int N, P;
  bool ok;
  __device__ __forceinline__ double2 load(int pos, int) const {
    const int o = offset_of(pos, N, P);
    if (!ok || o == kExcluded) return make_double2(0.0, 0.0);
    return __ldg(base + int64_t(o < 0 ? -o : o) * sp);
  }
};
struct FoldF {
  const double2* p;
  int64_t si, sk, sp;
  int N, P;
  __device__ __forceinline__ FoldAt at(int i, int k, bool ok) const {
    return FoldAt{p + i * si + k * sk, sp, N, P, ok};
  }
};

// Spectral multiply between the forward and inverse z transforms of pass C.  The folded
// octant values for this thread's first-stage slots are prefetched into registers (kv) before
// the forward transform starts, so their latency hides behind it.
template <int T>
struct SmemMulAt {
  static constexpr bool kSmem = true;
  const double2* sm;
  int t;
  const double2* kv;
  __device__ __forceinline__ double2 load(int pos, int e) const { return cmul(sm[tidx<T>(pos, t)], kv[e]); }
};
struct RegMulAt {
  static constexpr bool kSmem = false;
  const double2* v;
  const double2* kv;
  __device__ __forceinline__ double2 load(int, int e) const { return cmul(v[e], kv[e]); }
};
// Kernel-spectrum octant addressing for pass C lines (i = ky, k = kx; position kz):
// element = p + fold(kx) * s_kx + fold(ky) * s_ky + fold(kz) * s_kz.
// kx is the local spectral column of an x-slab: global kx = kx + kx_off (0 unsharded).
struct KOct {
  const double2* p;
  int Px, Py, Pz;
  int64_t s_kx, s_ky, s_kz;
  int kx_off;
  int quad = 0;  // pass-C line order of the persistent kernels: kx mirror pairs interleaved (1)
  int kx_base = 0;  // first folded kx row stored at p (x-slab kernels hold a row window)
  __device__ __forceinline__ const double2* line(int ky, int kx) const {
    return p + (fold_index(kx + kx_off, Px) - kx_base) * s_kx + fold_index(ky, Py) * s_ky;
  }
};

// ---------------------------------------------------------------------------- static plans
// Compile-time-planned kernels for the hot padded lengths (apply passes only; the one-off
// kernel-spectrum build uses the runtime-planned kernels).  Register budget: 64 per thread
// (minBlocks = 1024 threads / block size), i.e. 32 resident warps per SM.
template <class RL, int T>
struct SBounds {
  static constexpr int threads = RL::tpl() * T;
  static constexpr int min_blocks = threads >= 1024 ? 1 : 1024 / threads;
  // pass C keeps the forward spectrum and the prefetched K^ slots live: allow ~96 registers
  static constexpr int conv_min_blocks = threads >= 680 ? 1 : 680 / threads;
};

// Tile endpoints for the row side of transposing passes (staged through shared memory so the
// global access is line-major: 32 consecutive positions of one row per warp instruction).
template <int T>
struct TileIn {
  static constexpr bool kSmem = true;
  const double2* sm;
  int t, nvalid;
  __device__ __forceinline__ double2 load(int pos, int) const {
    return pos < nvalid ? sm[tidx<T>(pos, t)] : make_double2(0.0, 0.0);
  }
};

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const size_t ga = __cvta_generic_to_global(gmem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(ga), "r"(valid ? 16 : 0)
               : "memory");
}

// ROWIN: the input lines are contiguous rows (sp = 1): load the tile's valid rows line-major
// with cp.async, then transform from shared memory.  ROWOUT: the output lines are contiguous
// rows: the last stage writes the tile and the CTA stores it line-major.  Otherwise the first
// (last) stage reads (writes) global memory directly, T adjacent lines = T*16 contiguous bytes.
// compile-time choice between two endpoints (by reference)
template <bool C, class A, class B>
__device__ __forceinline__ auto& select_ref(A& a, B& b) {
  if constexpr (C) return a;
  else return b;
}

// LD is GLoadF for the apply passes, KGenF / FoldF for the kernel-spectrum build (ROWIN and
// ROWOUT need GLoadF / GStoreF).
template <class RL, int T, bool INV, bool ROWIN, bool ROWOUT, class LD = GLoadF>
__global__ void __launch_bounds__(SBounds<RL, T>::threads, SBounds<RL, T>::min_blocks)
    axis_pass_s(LineGeom g, LD ld, GStoreF st, const double2* __restrict__ tw) {
  static_assert(!ROWIN || std::is_same<LD, GLoadF>::value, "row-staged input needs a plain load");
  constexpr int NT = SBounds<RL, T>::threads;
  extern __shared__ double2 sm[];
  const int tile = blockIdx.x % g.ntiles;
  const int k = blockIdx.x / g.ntiles;
  const int t = threadIdx.x % T, jt = threadIdx.x / T;
  const int i = tile * T + t;
  const bool ok = i < g.n_inner;
  const int lines_ok = min(T, g.n_inner - tile * T);
  if constexpr (ROWIN) {
    const int nin = ld.g.nvalid;
    const double2* base = ld.g.p + int64_t(tile) * T * ld.g.si + k * ld.g.sk;
#pragma unroll
    for (int tt = 0; tt < T; ++tt)
      for (int pos = threadIdx.x; pos < nin; pos += NT)
        cp_async16_zfill(&sm[tidx<T>(pos, tt)], tt < lines_ok ? base + tt * ld.g.si + pos : ld.g.p,
                         tt < lines_ok);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  auto gsrc = ld.at(ok ? i : 0, k, ok);
  auto gdst = st.at(ok ? i : 0, k, ok);
  SmemIO<T> tdst{sm, t};
  auto src = [&]() {
    if constexpr (ROWIN) return TileIn<T>{sm, t, ld.g.nvalid};
    else return gsrc;
  }();
  auto& dst = select_ref<ROWOUT>(tdst, gdst);
  // twiddles staged in shared memory (first used after stage 1's barrier)
  double2* tws = sm + RL::len() * T;
  for (int m = threadIdx.x; m < RL::len(); m += NT) tws[m] = __ldg(tw + m);
  fft_line_s<RL, T, INV>(sm, t, jt, tws, src, dst);
  if constexpr (ROWOUT) {
    __syncthreads();
    const int nout = st.g.nvalid;
    double2* base = st.g.p + int64_t(tile) * T * st.g.si + k * st.g.sk;
    const double sc = st.g.scale;
#pragma unroll
    for (int tt = 0; tt < T; ++tt)
      if (tt < lines_ok)
        for (int pos = threadIdx.x; pos < nout; pos += NT) {
          const double2 v = sm[tidx<T>(pos, tt)];
          base[tt * st.g.si + pos] = (sc == 1.0) ? v : cscale(v, sc);
        }
  }
}

// K^ read straight from global memory at the multiply (no register prefetch).
struct RegMulGlobalAt {
  static constexpr bool kSmem = false;
  const double2* v;
  const double2* kline;
  int64_t sz;
  int P;
  bool ok;
  __device__ __forceinline__ double2 load(int pos, int e) const {
    return ok ? cmul(v[e], __ldg(kline + int64_t(fold_index(pos, P)) * sz)) : make_double2(0.0, 0.0);
  }
};

// MINB: min resident blocks (register cap); KPREF: prefetch K^ into registers first.
template <class RL, int T, int MINB, bool KPREF>
__global__ void __launch_bounds__(SBounds<RL, T>::threads, MINB)
    conv_pass_s(LineGeom g, GLoadF ld, GStoreF st, KOct ko, const double2* tw) {
  extern __shared__ double2 sm[];
  const int tile = blockIdx.x % g.ntiles;
  const int k = blockIdx.x / g.ntiles;  // ky
  const int t = threadIdx.x % T, jt = threadIdx.x / T;
  const int i = tile * T + t;           // kx
  const bool ok = i < g.n_inner;
  const int ii = ok ? i : 0;
  const double2* kline = ko.line(ii, k);
  const int64_t sz = ko.s_kz;
  double2 kv[kMaxElems];
  if constexpr (KPREF) {
#pragma unroll
    for (int e = 0; e < kMaxElems; ++e) {
      const int p = first_stage_pos_s<RL>(jt, e);
      kv[e] = (ok && p >= 0) ? __ldg(kline + int64_t(fold_index(p, RL::len())) * sz)
                             : make_double2(0.0, 0.0);
    }
  }
  auto src = ld.at(ii, k, ok);
  auto dst = st.at(ii, k, ok);
  double2* tws = sm + RL::len() * T;
  for (int m = threadIdx.x; m < RL::len(); m += SBounds<RL, T>::threads) tws[m] = __ldg(tw + m);
  tw = tws;
  if constexpr (RL::at(0) == RL::at(RL::n - 1)) {
    RegIO mid;
    fft_line_s<RL, T, false>(sm, t, jt, tw, src, mid);
    __syncthreads();
    if constexpr (KPREF) {
      RegMulAt msrc{mid.v, kv};
      fft_line_s<RL, T, true>(sm, t, jt, tw, msrc, dst);
    } else {
      RegMulGlobalAt msrc{mid.v, kline, sz, RL::len(), ok};
      fft_line_s<RL, T, true>(sm, t, jt, tw, msrc, dst);
    }
  } else {
    static_assert(KPREF, "smem hand-off variant prefetches K^");
    SmemIO<T> mid{sm, t};
    fft_line_s<RL, T, false>(sm, t, jt, tw, src, mid);
    __syncthreads();
    SmemMulAt<T> msrc{sm, t, kv};
    fft_line_s<RL, T, true>(sm, t, jt, tw, msrc, dst);
  }
}

using AxisFn = void (*)(LineGeom, GLoadF, GStoreF, const double2*);
using GenFn = void (*)(LineGeom, KGenF, GStoreF, const double2*);
using FoldFn = void (*)(LineGeom, FoldF, GStoreF, const double2*);
using ConvFn = void (*)(LineGeom, GLoadF, GStoreF, KOct, const double2*);

// One table per pass kind; per length the first entry is the default, FUSG_{ROW,COL,CONV}_VAR
// selects another (tuning knob).  Row passes (x: A, E) and column passes (y: B, D) share the
// axis kernels; conv is pass C.
struct StaticEntry {
  int L, T, threads;
  AxisFn fwd, inv;   // plain (strided global on both sides)
  ConvFn conv;
  AxisFn fwd_rowin, inv_rowout;  // transposing passes: row side staged line-major
  GenFn build_gen;                // kernel-spectrum build: generate K + forward (G1)
  FoldFn build_fold;              // even extension + forward (G2, G3)
};

#define FUSG_AX(TT, ...)                                                                   \
  StaticEntry {                                                                            \
    Radices<__VA_ARGS__>::len(), TT, Radices<__VA_ARGS__>::tpl() * TT,                     \
        axis_pass_s<Radices<__VA_ARGS__>, TT, false, false, false>,                          \
        axis_pass_s<Radices<__VA_ARGS__>, TT, true, false, false>, nullptr,                  \
        axis_pass_s<Radices<__VA_ARGS__>, TT, false, true, false>,                           \
        axis_pass_s<Radices<__VA_ARGS__>, TT, true, false, true>,                            \
        axis_pass_s<Radices<__VA_ARGS__>, TT, false, false, false, KGenF>,                   \
        axis_pass_s<Radices<__VA_ARGS__>, TT, false, false, false, FoldF>                    \
  }
#define FUSG_CV(TT, MINB, KPREF, ...)                                                      \
  StaticEntry {                                                                            \
    Radices<__VA_ARGS__>::len(), TT, Radices<__VA_ARGS__>::tpl() * TT, nullptr, nullptr,   \
        conv_pass_s<Radices<__VA_ARGS__>, TT, MINB, KPREF>, nullptr, nullptr, nullptr, nullptr \
  }

enum StaticKind { kKindRow = 0, kKindCol = 1, kKindConv = 2 };

// generated ladder (static_gen.cpp): every entry of every generated TU, by kind
const StaticEntry* generated_static(int kind, size_t* n);

}  // namespace fusg
