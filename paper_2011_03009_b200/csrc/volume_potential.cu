// Volume-potential operator on the device: GreenKernel construction ("Evaluate G_k") and
// GreenKernel::apply (src/potential.cpp:72-151) as pruned, fused FP64 Stockham passes.
//
// apply(f) = crop_N( IDFT_P( K^ . DFT_P( pad_P(f) ) ) ) / |P|   (src/potential.cpp:128-149)
//
//   pass A  forward x : f [Nz][Ny][Nx]      -> A [Nz][Ny][Px]   (zero padding fused: rows of Nx)
//   pass B  forward y : A                    -> B [Nz][Py][Px]   (pruned input: Ny of Py)
//   pass C  forward z, * K^, inverse z: B -> B in place          (pruned in/out: Nz of Pz)
//   pass D  inverse y : B                    -> A               (pruned output: Ny)
//   pass E  inverse x, * scale/|P|, crop : A -> u [Nz][Ny][Nx]
//
// The padded kernel tensor is even along every axis (K[P-m] = K[m], offset_of at :88-94),
// so its spectrum is even too: only the octant [0,Px/2]x[0,Py/2]x[0,Pz/2] is built and
// stored, and pass C folds its index.  The octant is built by the same pass machinery with
// the kernel values generated in registers (no padded tensor is ever materialised).
#include <string>
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cstdio>
#include <vector>
#include <utility>

#include "internal.hpp"
#include "static_kernels.cuh"
#include "warp_args.cuh"

namespace fusg {

// ---------------------------------------------------------------------------- kernels
template <bool INV, int T, class LD, class ST>
__global__ void __launch_bounds__(512, 2) axis_pass(AxisPlan pl, LineGeom g, LD ld, ST st) {
  extern __shared__ double2 sm[];
  const int tile = blockIdx.x % g.ntiles;
  const int k = blockIdx.x / g.ntiles;
  const int t = threadIdx.x % T, jt = threadIdx.x / T;
  const int i = tile * T + t;
  const bool ok = i < g.n_inner;
  auto src = ld.at(ok ? i : 0, k, ok);
  auto dst = st.at(ok ? i : 0, k, ok);
  fft_line<INV, T>(pl, sm, t, jt, src, dst);
}

template <int T>
__global__ void __launch_bounds__(512, 2) conv_pass(AxisPlan pl, LineGeom g, GLoadF ld, GStoreF st,
                                                 KOct ko, int fuse_regs) {
  extern __shared__ double2 sm[];
  const int tile = blockIdx.x % g.ntiles;
  const int k = blockIdx.x / g.ntiles;  // ky
  const int t = threadIdx.x % T, jt = threadIdx.x / T;
  const int i = tile * T + t;           // kx
  const bool ok = i < g.n_inner;
  const int ii = ok ? i : 0;
  const double2* kline = ko.line(ii, k);
  double2 kv[kMaxElems];
#pragma unroll
  for (int e = 0; e < kMaxElems; ++e) {
    const int p = first_stage_pos(pl, jt, e);
    kv[e] = (ok && p >= 0) ? __ldg(kline + fold_index(p, ko.Pz) * ko.s_kz) : make_double2(0.0, 0.0);
  }
  auto src = ld.at(ii, k, ok);
  auto dst = st.at(ii, k, ok);
  if (fuse_regs) {
    // last forward radix == first inverse radix: the spectrum never leaves registers
    RegIO mid;
    fft_line<false, T>(pl, sm, t, jt, src, mid);
    __syncthreads();
    RegMulAt msrc{mid.v, kv};
    fft_line<true, T>(pl, sm, t, jt, msrc, dst);
  } else {
    SmemIO<T> mid{sm, t};
    fft_line<false, T>(pl, sm, t, jt, src, mid);
    __syncthreads();
    SmemMulAt<T> msrc{sm, t, kv};
    fft_line<true, T>(pl, sm, t, jt, msrc, dst);
  }
}

// ---------------------------------------------------------------------------- planning
static bool smooth7(int n) {
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) n /= p;
  return n == 1;
}

int smooth_padded_size(int n, bool pad_small_primes) {
  // Reference: 2N, or next_fast_size(2N) (src/potential.cpp:74-77). Any P >= 2N-1 gives
  // the same discrete operator; the device path needs {2,3,5,7}-smooth lengths.
  int p = pad_small_primes ? 2 * n : std::max(2, 2 * n - 1);
  while (!smooth7(p)) ++p;
  return p;
}

// Padded length the device uses on axis `axis`.  Any P >= 2N-1 is exact (offset_of,
// src/potential.cpp:88-94).  Every axis rounds up to the smallest length with compile-time
// planned kernels (hand-tuned tables + the generated ladder, gaps <= 12.5%): the runtime-planned
// kernels are ~2.6x slower.  Pz only lives inside pass C (which reads and writes the Nz valid
// values of each z-row) and the K^ octant, so on z the smallest length the persistent warp
// pass C covers (256, 512, 768, 1024) is preferred when within 1.35x: e.g. Nz = 323 runs pass C
// at 768 instead of the CTA-tiled kernel at 648.  FUSG_PZ_WARP=0 / FUSG_PAD_STATIC=0 disable.
static const std::vector<int>& static_lengths(bool conv);
int device_padded_size(int n, int axis) {
  const int smooth = smooth_padded_size(n, false);
  static const bool use_static = [] {  // FUSG_PAD_STATIC=0: smallest smooth size
    const char* e = getenv("FUSG_PAD_STATIC");
    return !(e && atoi(e) == 0);
  }();
  static const int pz_warp = [] {  // FUSG_PZ_WARP: 0 off, else the largest preferred length
    const char* e = getenv("FUSG_PZ_WARP");
    return e ? atoi(e) : 2048;
  }();
  int p = smooth;  // round up to a length with compile-time-planned kernels
  if (use_static)
    for (int L : static_lengths(axis == 2))
      if (L >= 2 * n - 1) {
        if (L <= smooth * 1.35) p = L;
        break;
      }
  static const int pxy_warp = [] {  // FUSG_PXY_WARP: prefer warp-engine lengths on x / y too
    const char* e = getenv("FUSG_PXY_WARP");
    return e ? atoi(e) : 0;
  }();
  if (axis != 2 && pxy_warp) {
    for (int L : {256, 512, 768, 1024, 1536})
      if (L <= pxy_warp && L >= 2 * n - 1) return (L <= p * 1.35) ? L : p;
    return p;
  }
  // x / y: the lengths with warp-transform transposing passes (512: 16x16x2; 1024, 1536: 2 / 3 x
  // 512 with TMA tiles) when within FUSG_PXY_FAST (default 1.06) of the static length: cfg3's
  // y 980 -> 1024 (passes B / D 4.8 -> ~2.5 ms)
  static const double pxy_fast = [] {
    const char* e = getenv("FUSG_PXY_FAST");
    return e ? atof(e) : 1.06;
  }();
  if (axis != 2 && pxy_fast > 1.0) {
    for (int L : {512, 1024, 1536})
      if (L >= 2 * n - 1) return (L > p && L <= p * pxy_fast) ? L : p;
    return p;
  }
  if (axis != 2 || !pz_warp) return p;
  for (int L : {256, 512, 768, 1024, 1536, 2048})  // persistent pass C (warp / multi-warp lines)
    if (L <= pz_warp && L >= 2 * n - 1) return (L <= p * 1.35) ? L : p;
  return p;
}

bool make_plan_radices(int L, AxisPlan& pl) {
  int m = L, e2 = 0, e3 = 0, e5 = 0, e7 = 0;
  while (m % 2 == 0) { m /= 2; ++e2; }
  while (m % 3 == 0) { m /= 3; ++e3; }
  while (m % 5 == 0) { m /= 5; ++e5; }
  while (m % 7 == 0) { m /= 7; ++e7; }
  if (m != 1 || L < 2) return false;
  std::vector<int> r;
  if (e2 > 0) {
    const int n = (e2 + 2) / 3;  // stages for the power of two, <= 3 bits each, balanced
    for (int s = 0; s < n; ++s) {
      const int bits = e2 / n + (s < e2 % n ? 1 : 0);
      r.push_back(1 << bits);
    }
  }
  for (int i = 0; i < e7; ++i) r.push_back(7);
  for (int i = 0; i < e5; ++i) r.push_back(5);
  for (int i = 0; i < e3; ++i) r.push_back(3);
  // Put a repeated radix (largest first) at both ends: pass C then hands the forward
  // spectrum to the inverse transform in registers (first/last radix equal).
  std::sort(r.begin(), r.end(), [](int a, int b) { return a > b; });
  for (size_t a = 0; a + 1 < r.size(); ++a) {
    if (r[a] == r[a + 1]) {
      const int rv = r[a];
      r.erase(r.begin() + a, r.begin() + a + 2);
      r.insert(r.begin(), rv);
      r.push_back(rv);
      break;
    }
  }
  if (int(r.size()) > kMaxStages) return false;
  pl.L = L;
  pl.nst = int(r.size());
  int ns = 1, tpl = 1;
  for (int s = 0; s < pl.nst; ++s) {
    pl.radix[s] = r[s];
    pl.ns[s] = ns;
    ns *= r[s];
    const int nb = L / r[s];
    const int bmax = kMaxElems / r[s];
    tpl = std::max(tpl, (nb + bmax - 1) / bmax);
  }
  pl.tpl = tpl;
  return true;
}

static fusg_status upload_twiddles(fusg_ctx* ctx, int L, double2** out) {
  std::lock_guard<std::mutex> lock(ctx->tw_mu);
  auto it = ctx->tw_cache.find(L);
  if (it != ctx->tw_cache.end()) {
    *out = it->second;
    return FUSG_OK;
  }
  std::vector<double2> h(L);
  for (int m = 0; m < L; ++m) {
    // exp(-2 pi i m / L) with the angle reduced to the first octant for accuracy
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * m / L;
    h[m] = make_double2(double(cosl(a)), double(sinl(a)));
  }
  FUSG_CUDA_TRY(cudaMalloc(out, sizeof(double2) * L));
  FUSG_CUDA_TRY(cudaMemcpy(*out, h.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
  ctx->tw_cache[L] = *out;
  return FUSG_OK;
}

constexpr size_t kSmemBudget = 100 * 1024;

static int choose_tile(const AxisPlan& pl, int n_inner) {
  int T = 16;
  while (T > 1 && (size_t(pl.L) * T * sizeof(double2) > kSmemBudget || T * pl.tpl > 512 ||
                   (T / 2 >= n_inner)))
    T /= 2;
  return T;
}

static const StaticEntry kRowTab[] = {
    FUSG_AX(4, 8, 8, 8),        // 512  (cfg2)
    FUSG_AX(8, 8, 8, 8),
    FUSG_AX(16, 4, 8, 4),       // 128  (cfg1)
    FUSG_AX(4, 8, 4, 3, 8),     // 768
    FUSG_AX(8, 8, 4, 3, 8),
    FUSG_AX(4, 8, 4, 4, 8),     // 1024 (pass C runs the warp kernel; build G3 and x/y here)
    FUSG_AX(4, 8, 8, 3, 8),     // 1536 (cfg5): 64 B column segments (T = 2 measured 15% slower)
    FUSG_AX(2, 8, 8, 3, 8),
    FUSG_AX(2, 5, 7, 3, 2, 5),  // 1050 (cfg3 x)
    FUSG_AX(2, 7, 4, 5, 7),     // 980  (cfg3 y, z)
    FUSG_AX(4, 5, 5, 5, 5),     // 625  (desk cfg4)
    FUSG_AX(4, 3, 8, 3, 3, 3),  // 648  (desk cfg4)
    FUSG_AX(4, 8, 7, 4, 3),     // 672  (desk cfg4)
};
static const StaticEntry kColTab[] = {
    FUSG_AX(8, 8, 8, 8),
    FUSG_AX(4, 8, 8, 8),
    FUSG_AX(16, 4, 8, 4),
    FUSG_AX(4, 8, 4, 3, 8),
    FUSG_AX(8, 8, 4, 3, 8),
    FUSG_AX(4, 8, 4, 4, 8),
    FUSG_AX(4, 8, 8, 3, 8),
    FUSG_AX(2, 8, 8, 3, 8),
    FUSG_AX(2, 5, 7, 3, 2, 5),
    FUSG_AX(2, 7, 4, 5, 7),
    FUSG_AX(4, 5, 5, 5, 5),
    FUSG_AX(4, 3, 8, 3, 3, 3),
    FUSG_AX(4, 8, 7, 4, 3),
};
static const StaticEntry kConvTab[] = {
    FUSG_CV(8, 1, true, 8, 8, 8),
    FUSG_CV(4, 3, true, 8, 8, 8),
    FUSG_CV(4, 4, false, 8, 8, 8),
    FUSG_CV(8, 2, false, 8, 8, 8),
    FUSG_CV(4, 2, true, 8, 8, 8),
    FUSG_CV(16, 1, true, 4, 8, 4),
    FUSG_CV(4, 1, true, 8, 8, 3, 8),
    FUSG_CV(2, 1, true, 8, 8, 3, 8),
    FUSG_CV(2, 1, true, 5, 7, 3, 2, 5),
    FUSG_CV(2, 1, true, 7, 4, 5, 7),
    FUSG_CV(4, 1, true, 5, 5, 5, 5),
    FUSG_CV(4, 1, true, 3, 8, 3, 3, 3),
    FUSG_CV(4, 1, true, 8, 7, 4, 3),
};


// FUSG_STATIC=0 disables the compile-time-planned kernels.
static const StaticEntry* find_static(int L, int kind) {
  static const bool enabled = [] {
    const char* e = getenv("FUSG_STATIC");
    return !(e && atoi(e) == 0);
  }();
  static const int var[3] = {
      getenv("FUSG_ROW_VAR") ? atoi(getenv("FUSG_ROW_VAR")) : 0,
      getenv("FUSG_COL_VAR") ? atoi(getenv("FUSG_COL_VAR")) : 0,
      getenv("FUSG_CONV_VAR") ? atoi(getenv("FUSG_CONV_VAR")) : 0};
  if (!enabled) return nullptr;
  const StaticEntry* tab = kind == kKindRow ? kRowTab : kind == kKindCol ? kColTab : kConvTab;
  const size_t n = kind == kKindRow ? sizeof(kRowTab) / sizeof(StaticEntry)
                   : kind == kKindCol ? sizeof(kColTab) / sizeof(StaticEntry)
                                      : sizeof(kConvTab) / sizeof(StaticEntry);
  const StaticEntry* first = nullptr;
  int seen = 0;
  for (size_t q = 0; q < n; ++q) {
    if (tab[q].L != L) continue;
    if (!first) first = &tab[q];
    if (seen++ == var[kind]) return &tab[q];
  }
  if (first) return first;
  size_t ng = 0;  // generated ladder (tools/gen_static.py)
  const StaticEntry* gen = generated_static(kind, &ng);
  for (size_t q = 0; q < ng; ++q)
    if (gen[q].L == L) return &gen[q];
  return nullptr;
}

// Padded lengths with compile-time-planned kernels, ascending: axis = row and column kernels
// (x, y), conv = pass C (z).
static const std::vector<int>& static_lengths(bool conv) {
  static const std::vector<int> lens[2] = {[] {
    std::vector<int> v, out;
    for (const auto& e : kRowTab) v.push_back(e.L);
    size_t ng = 0;
    const StaticEntry* gen = generated_static(kKindRow, &ng);
    for (size_t q = 0; q < ng; ++q) v.push_back(gen[q].L);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    for (int L : v)
      if (find_static(L, kKindRow) && find_static(L, kKindCol)) out.push_back(L);
    return out;
  }(), [] {
    std::vector<int> v;
    for (const auto& e : kConvTab) v.push_back(e.L);
    size_t ng = 0;
    const StaticEntry* gen = generated_static(kKindConv, &ng);
    for (size_t q = 0; q < ng; ++q) v.push_back(gen[q].L);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
  }()};
  return lens[conv ? 1 : 0];
}

}  // namespace fusg

extern "C" int32_t fusg_static_lengths(int32_t conv, int32_t* out, int32_t cap) {
  const auto& v = fusg::static_lengths(conv != 0);
  for (int32_t i = 0; out && i < cap && i < int32_t(v.size()); ++i) out[i] = v[size_t(i)];
  return int32_t(v.size());
}

namespace fusg {
// ---------------------------------------------------------------------------- warp engine
// Warp-per-line kernels (fft_warp.cuh) for L <= 512: rows (x passes) are read and written
// straight from global memory by their own lane group; columns (y, z passes) are staged as a
// swizzled [pos][8] tile with one coalesced cooperative load and store (2 CTA barriers per
// tile), the transforms in between use __syncwarp only.


constexpr int kWarpThreads = 256;  // 8 warps per CTA
#ifndef FUSG_WARP_MINB
#define FUSG_WARP_MINB 2  // resident CTAs per SM the register budget is sized for
#endif

// Transposing passes on the warp engine.  A CTA owns 8 adjacent lines (i0..i0+7 at outer k); warp w
// transforms line w using column w of a swizzled [pos][8] shared tile as its exchange buffer.
//   row_to_col: input rows are contiguous (sp = 1): each warp loads its own row (512 B per warp
//               instruction); the last stage writes the tile; after one barrier the CTA stores
//               positions as 8 adjacent lines = 128 contiguous bytes (si = 1).
//   col_to_row: the mirror: a cooperative 128-byte-row load of the tile, one barrier, then each
//               warp transforms its column and stores its row contiguously.
template <class RL, bool INV, bool PRUNED>
__global__ void __launch_bounds__(kWarpThreads, 2) warp_row_to_col(WArgs a) {
  constexpr int E = RL::len() / 32;
  extern __shared__ double2 tile[];
  const int ntiles = (a.n_inner + 7) / 8;
  const int i0 = (blockIdx.x % ntiles) * 8;
  const int k = blockIdx.x / ntiles;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lines_ok = min(8, a.n_inner - i0);
  const bool ok = w < lines_ok;
  RowIn src{a.in + int64_t(i0 + (ok ? w : 0)) * a.in_si + int64_t(k) * a.in_sk, 1, a.in_nvalid, ok};
  TileEx ex{tile, w};
  TileColOut dst{tile, w};
  double2 v[E];
  warp_fft<RL, 32, INV, PRUNED ? 1 : 0>(v, ex, lane, TwTable{a.tw}, src, dst);  // PRUNED: nvalid <= L/2
  __syncthreads();
  if (a.pm.n == 0) {
    double2* base = a.out + int64_t(i0) * a.out_si + int64_t(k) * a.out_sk;
    for (int e = threadIdx.x; e < a.out_nvalid * 8; e += kWarpThreads) {
      const int pos = e >> 3, t = e & 7;
      if (t < lines_ok) {
        const double2 x = tile[tile_at(pos, t)];
        base[t * a.out_si + pos * a.out_sp] = (a.scale == 1.0) ? x : cscale(x, a.scale);
      }
    }
  } else {
    // fused transpose: the segment of position pos (kx) goes straight to the rank owning it
    for (int e = threadIdx.x; e < a.out_nvalid * 8; e += kWarpThreads) {
      const int pos = e >> 3, t = e & 7;
      if (t < lines_ok) {
        const int q = a.pm.owner(a.pm.by_pos ? pos : i0 + t);
        const double2 x = tile[tile_at(pos, t)];
        a.pm.base[q][a.pm.off[q] + int64_t(i0 + t) * a.out_si + int64_t(k) * a.pm.sk[q] + int64_t(pos) * a.out_sp] =
            (a.scale == 1.0) ? x : cscale(x, a.scale);
      }
    }
    __threadfence_system();  // remote stores performed before the barrier that follows the pass
  }
}

template <class RL, bool INV, bool PRUNED>
__global__ void __launch_bounds__(kWarpThreads, 2) warp_col_to_row(WArgs a) {
  constexpr int E = RL::len() / 32;
  extern __shared__ double2 tile[];
  const int ntiles = (a.n_inner + 7) / 8;
  const int i0 = (blockIdx.x % ntiles) * 8;
  const int k = blockIdx.x / ntiles;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lines_ok = min(8, a.n_inner - i0);
  const double2* base = a.in + int64_t(i0) * a.in_si + int64_t(k) * a.in_sk;
  for (int e = threadIdx.x; e < a.in_nvalid * 8; e += kWarpThreads) {
    const int pos = e >> 3, t = e & 7;
    tile[tile_at(pos, t)] = t < lines_ok ? __ldg(base + t * a.in_si + pos * a.in_sp) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const bool ok = w < lines_ok;
  TileColIn src{tile, w, a.in_nvalid};
  TileEx ex{tile, w};
  RowOut dst{a.out + int64_t(i0 + (ok ? w : 0)) * a.out_si + int64_t(k) * a.out_sk, 1, a.out_nvalid, ok,
             a.scale};
  double2 v[E];
  warp_fft<RL, 32, INV, PRUNED ? 2 : 0>(v, ex, lane, TwTable{a.tw}, src, dst);  // PRUNED: nout <= L/2
}

// Passes D/E, persistent: one CTA of 8 warps per SM streams 8-line column tiles ([pos][8],
// swizzled) with cp.async double buffering.  Tile i+1 is in flight while warp w transforms line
// w of tile i in place (its column of the tile, __syncwarp only) and writes its output row
// straight from registers (512 B per warp instruction).  Two CTA barriers per tile.
template <class RL, bool PRUNED>
__global__ void __launch_bounds__(kWarpThreads, 1) warp_col_to_row_pp(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / 32;
  extern __shared__ double2 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles_i = (a.n_inner + 7) / 8;
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto buf = [&](int b) { return sm + b * (L * 8); };
  auto prefetch = [&](int64_t tix, int b) {
    if (tix < ntiles) {
      const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * 8;
      const int k = int(unsigned(tix) / unsigned(ntiles_i));
      const int lines_ok = min(8, a.n_inner - i0);
      const double2* base = a.in + int64_t(i0) * a.in_si + int64_t(k) * a.in_sk;
      double2* t = buf(b);
      for (int e = threadIdx.x; e < a.in_nvalid * 8; e += kWarpThreads) {
        const int pos = e >> 3, tt = e & 7;
        cp_async16_zfill(&t[tile_at(pos, tt)], tt < lines_ok ? base + tt * a.in_si + pos * a.in_sp : a.in,
                         tt < lines_ok);
      }
    }
    cp_async_commit();
  };
  int64_t tix = blockIdx.x;
  prefetch(tix, 0);
  for (int it = 0; tix < ntiles; tix += gridDim.x, ++it) {
    const int b = it & 1;
    __syncthreads();  // every warp is done with the other buffer (the previous tile)
    prefetch(tix + gridDim.x, b ^ 1);
    cp_async_wait1();
    __syncthreads();  // this tile's copies (issued by all threads) have landed
    const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * 8;
    const int k = int(unsigned(tix) / unsigned(ntiles_i));
    const bool ok = w < min(8, a.n_inner - i0);
    double2* const t = buf(b);
    TileColIn src{t, w, a.in_nvalid};
    TileEx ex{t, w};
    const int line = i0 + (ok ? w : 0);
    double2* orow = a.out + int64_t(line) * a.out_si + int64_t(k) * a.out_sk;
    if (a.pm.n) {  // fused transpose: the row goes straight to the rank owning line (z)
      const int q = a.pm.owner(line);
      orow = a.pm.base[q] + (a.pm.off[q] + int64_t(line) * a.out_si + int64_t(k) * a.pm.sk[q]);
    }
    RowOut dst{orow, 1, a.out_nvalid, ok, a.scale};
    double2 v[E];
    warp_fft<RL, 32, true, PRUNED ? 2 : 0>(v, ex, lane, TwTable{a.tw}, src, dst);  // PRUNED: nout <= L/2
  }
  cp_async_wait0();
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

// Lines (i, k), i fastest: consecutive lane groups of a CTA take consecutive i, so column
// lines (position stride sp, i contiguous) from one CTA share every 128-byte row through L1.
template <class RL, int LANES, bool INV>
__global__ void __launch_bounds__(kWarpThreads, FUSG_WARP_MINB) warp_line_pass(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int LPC = kWarpThreads / LANES;  // lines per CTA
  extern __shared__ double2 sm[];
  const int g = threadIdx.x / LANES, lane = threadIdx.x % LANES;
  const int64_t line = int64_t(blockIdx.x) * LPC + g;
  const bool ok = line < int64_t(a.n_inner) * a.n_outer;
  const int64_t li = ok ? line : 0;
  const int64_t i = li % a.n_inner, k = li / a.n_inner;
  PrivEx ex{sm + g * L};
  RowIn src{a.in + i * a.in_si + k * a.in_sk, a.in_sp, a.in_nvalid, ok};
  RowOut dst{a.out + i * a.out_si + k * a.out_sk, a.out_sp, a.out_nvalid, ok, a.scale};
  double2 v[E];
  warp_fft<RL, LANES, INV>(v, ex, lane, TwTable{a.tw}, src, dst);
}


// Pass C on rows of B [kx][ky][z] (z contiguous): forward z, * K^ (octant row [kx][ky][kz],
// contiguous), inverse z; in place.  n_inner = Py, n_outer = Px.
template <class RL, int LANES>
__global__ void __launch_bounds__(kWarpThreads, FUSG_WARP_MINB) warp_row_conv(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int LPC = kWarpThreads / LANES;
  static_assert(RL::at(0) == RL::at(RL::n - 1), "register hand-off needs equal first/last radix");
  extern __shared__ double2 sm[];
  const int g = threadIdx.x / LANES, lane = threadIdx.x % LANES;
  const int64_t line = int64_t(blockIdx.x) * LPC + g;
  const bool ok = line < int64_t(a.n_inner) * a.n_outer;
  const int64_t li = ok ? line : 0;
  const int ky = interleave_index(int(li % a.n_inner), a.ko.Py);
  // mirror-interleave kx only when this launch owns every column (unsharded)
  const int kx = a.n_outer == a.ko.Px ? interleave_index(int(li / a.n_inner), a.ko.Px)
                                      : int(li / a.n_inner);
  const double2* kline = a.ko.line(ky, kx);
  PrivEx ex{sm + g * L};
  RowIn src{a.in + ky * a.in_si + int64_t(kx) * a.in_sk, 1, a.in_nvalid, ok};
  double2 v[E];
  RegsOut mid{v};
  warp_fft<RL, LANES, false>(v, ex, lane, TwTable{a.tw}, src, mid);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int pos = in_pos<RL, LANES, 0>(lane, e);
    v[e] = cmul(v[e], __ldg(kline + fold_index(pos, L)));
  }
  RegsIn msrc{v};
  RowOut dst{a.out + ky * a.out_si + int64_t(kx) * a.out_sk, 1, a.out_nvalid, ok, a.scale};
  warp_fft<RL, LANES, true>(v, ex, lane, TwTable{a.tw}, msrc, dst);
}

// Pass C, persistent and software-pipelined: every warp streams lines (stride = all warps of
// the grid).  Per warp, shared memory holds an exchange buffer X (L), an input staging buffer S
// (L/2 when PRUNED: the zero-padded half is never staged) and the K^ row.  S and the K^ row are
// single-buffered: the next line's input is copied into S (cp.async) as soon as the first
// forward stage has read it into registers, and the next K^ row right after the spectral
// multiply, so both copies overlap the rest of the line's transform without a second buffer.
// The small footprint (~16 KB per warp) lets 12 warps share an SM.  No CTA barriers.


// BULK: the input row and the K^ row are staged by one lane's 1-D bulk copy (TMA) into linear
// buffers, completion tracked by the warp's two mbarriers; else by per-lane cp.async into a
// swizzled S (measured: the LDGSTS path costs 2.4x its ideal shared wavefronts).
template <class RL, int LANES, bool PRUNED, bool BULK>
__global__ void __launch_bounds__(kPPWarps * 32, pp_min_blocks<RL::len()>()) warp_row_conv_pp(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int HZ = L / 2 + 1;
  constexpr int R0 = RL::at(0);
  using SM = PPConvSmem<L, PRUNED>;
  static_assert(LANES == 32, "one line per warp");
  static_assert(RL::at(0) == RL::at(RL::n - 1), "register hand-off needs equal first/last radix");
  extern __shared__ double2 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // buffers addressed arithmetically from the shared base (a runtime-indexed pointer array
  // would demote every access to generic LD/ST)
  double2* const xb = sm + size_t(w) * SM::PER_WARP;
  double2* const sb = xb + L;
  double2* const kb = sb + SM::STAGE;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + size_t(kPPWarps) * SM::PER_WARP) + 2 * w;
  if constexpr (BULK) {
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      mbar_init_fence();
    }
    __syncwarp();
  }
  unsigned ph_in = 0, ph_k = 0;
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t stride = int64_t(gridDim.x) * kPPWarps;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) {
    conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx);
  };
  // staged position p lives at S[swz(p)] (PRUNED: p < L/2, so the swizzle stays inside S)
  // (each line's (ky, kx) -- ~45 instructions of divisions -- is computed once, one line ahead, and
  // serves both refills and the output row)
  auto prefetch_in = [&](bool ok, int ky, int kx) {
    if (ok) {
      const double2* in = a.in + ky * a.in_si + int64_t(kx) * a.in_sk;
      if constexpr (BULK) {
        if (lane == 0) bulk_stage(sb, in, unsigned(a.in_nvalid) * sizeof(double2), bars);
      } else {
        for (int pos = lane; pos < a.in_nvalid; pos += 32) cp_async16(sb + swz(pos), in + pos);
      }
    }
    if constexpr (!BULK) cp_async_commit();
  };
  auto prefetch_k = [&](bool ok, int ky, int kx) {
    if (ok) {
      const double2* kl = a.ko.line(ky, kx);
      if constexpr (BULK) {
        if (lane == 0) bulk_stage(kb, kl, HZ * sizeof(double2), bars + 1);
      } else {
        for (int kz = lane; kz < HZ; kz += 32) cp_async16(kb + kz, kl + kz);
      }
    }
    if constexpr (!BULK) cp_async_commit();
  };
  const TwTable tw{a.tw};
  // PRUNED (host-selected when Nz <= L/2): zero-padded input and cropped output halves run the
  // pruned first forward and last inverse radix-8 stages
  constexpr int kPin = PRUNED ? 1 : 0, kPout = PRUNED ? 2 : 0;
  const PrivEx ex{xb};
  int64_t line = int64_t(blockIdx.x) * kPPWarps + w;
  int ky = 0, kx = 0;
  if (line < nlines) coords(line, ky, kx);
  prefetch_in(line < nlines, ky, kx);
  prefetch_k(line < nlines, ky, kx);
  for (; line < nlines; line += stride) {
    const bool more = line + stride < nlines;
    int kyn = 0, kxn = 0;
    if (more) coords(line + stride, kyn, kxn);
    if constexpr (BULK) {
      mbar_wait(bars, ph_in);  // this line's staged input has landed
      ph_in ^= 1;
    } else {
      cp_async_wait0();
      __syncwarp();  // this line's staged input and K^ row are visible to the whole warp
    }
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((PRUNED && R0 == 8) && (e % R0) >= R0 / 2) continue;  // zero padding: not staged
      const int pos = in_pos<RL, LANES, 0>(lane, e);
      v[e] = pos < a.in_nvalid ? sb[BULK ? pos : swz(pos)] : make_double2(0.0, 0.0);
    }
    __syncwarp();  // S consumed: refill it with the next line while this one is transformed
    prefetch_in(more, kyn, kxn);
    RegsIn vin{v};
    RegsOut mid{v};
    warp_fft<RL, LANES, false, kPin>(v, ex, lane, tw, vin, mid);
    if constexpr (BULK) {
      mbar_wait(bars + 1, ph_k);  // this line's K^ row has landed
      ph_k ^= 1;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = cmul(v[e], kb[fold_index(in_pos<RL, LANES, 0>(lane, e), L)]);
    __syncwarp();  // K^ row consumed
    prefetch_k(more, kyn, kxn);
    RowOut dst{a.out + ky * a.out_si + int64_t(kx) * a.out_sk, 1, a.out_nvalid, true, a.scale};
    ky = kyn;
    kx = kxn;
    warp_fft<RL, LANES, true, kPout>(v, ex, lane, tw, vin, dst);
  }
  if constexpr (!BULK) cp_async_wait0();
}

using WFn = void (*)(WArgs);

template <class RL>
constexpr bool whole_butterflies(int lanes) {
  const int E = RL::len() / lanes;
  if (RL::len() % lanes) return false;
  for (int s = 0; s < RL::n; ++s)
    if (E % RL::at(s)) return false;
  return true;
}
// Pass C on multi-warp lines: the persistent pipeline of warp_row_conv_pp with each line owned
// by a group of LANES = 64..256 lanes (2..8 warps); the exchanges synchronise the group with a
// named barrier.  GROUPS line groups per CTA, MINB CTAs per SM for the register budget.  Long
// lines (1536, 2048) need it for registers; short ones (512, 1024) use it to put more warps on
// each line in flight (latency hiding at the same shared-memory footprint).
template <int L, bool PRUNED, int GROUPS>
struct PP64Smem {
  static constexpr int KROW = ((L / 2 + 1) + 1) & ~1;
  static constexpr int STAGE = PRUNED ? L / 2 : L;
  static constexpr int PER_GROUP = L + STAGE + KROW;
  static constexpr size_t BYTES = size_t(GROUPS) * PER_GROUP * sizeof(double2) + GROUPS * 2 * sizeof(uint64_t);
};

template <class RL, int LANES, int GROUPS, int MINB, bool PRUNED, bool BULK>
__global__ void __launch_bounds__(GROUPS * LANES, MINB) warp_row_conv_pp64(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int HZ = L / 2 + 1;
  constexpr int R0 = RL::at(0);
  using SM = PP64Smem<L, PRUNED, GROUPS>;
  static_assert(GROUPS < 16, "named barrier ids 1..15");
  static_assert(RL::at(0) == RL::at(RL::n - 1), "register hand-off needs equal first/last radix");
  extern __shared__ double2 sm[];
  const int grp = threadIdx.x / LANES, lane = threadIdx.x % LANES;
  const GroupSync<LANES> sync{1 + grp};
  double2* const xb = sm + size_t(grp) * SM::PER_GROUP;
  double2* const sb = xb + L;
  double2* const kb = sb + SM::STAGE;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + size_t(GROUPS) * SM::PER_GROUP) + 2 * grp;
  if constexpr (BULK) {
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      mbar_init_fence();
    }
    sync();
  }
  unsigned ph_in = 0, ph_k = 0;
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t stride = int64_t(gridDim.x) * GROUPS;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) {
    conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx);
  };
  auto prefetch_in = [&](int64_t line) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      const double2* in = a.in + ky * a.in_si + int64_t(kx) * a.in_sk;
      if constexpr (BULK) {
        if (lane == 0) bulk_stage(sb, in, unsigned(a.in_nvalid) * sizeof(double2), bars);
      } else {
        for (int pos = lane; pos < a.in_nvalid; pos += LANES) cp_async16(sb + swz(pos), in + pos);
      }
    }
    if constexpr (!BULK) cp_async_commit();
  };
  auto prefetch_k = [&](int64_t line) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      const double2* kl = a.ko.line(ky, kx);
      if constexpr (BULK) {
        if (lane == 0) bulk_stage(kb, kl, HZ * sizeof(double2), bars + 1);
      } else {
        for (int kz = lane; kz < HZ; kz += LANES) cp_async16(kb + kz, kl + kz);
      }
    }
    if constexpr (!BULK) cp_async_commit();
  };
  const TwTable tw{a.tw};
  constexpr int kPin = PRUNED ? 1 : 0, kPout = PRUNED ? 2 : 0;
  const PrivEx ex{xb};
  int64_t line = int64_t(blockIdx.x) * GROUPS + grp;
  prefetch_in(line);
  prefetch_k(line);
  for (; line < nlines; line += stride) {
    if constexpr (BULK) {
      mbar_wait(bars, ph_in);  // the group's staged input has landed
      ph_in ^= 1;
    } else {
      cp_async_wait0();
      sync();  // the group's staged input and K^ row have landed
    }
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((PRUNED && R0 == 8) && (e % R0) >= R0 / 2) continue;
      const int pos = in_pos<RL, LANES, 0>(lane, e);
      v[e] = pos < a.in_nvalid ? sb[BULK ? pos : swz(pos)] : make_double2(0.0, 0.0);
    }
    sync();  // staging consumed by the whole group
    prefetch_in(line + stride);
    RegsIn vin{v};
    RegsOut mid{v};
    warp_fft<RL, LANES, false, kPin>(v, ex, lane, tw, vin, mid, sync);
    if constexpr (BULK) {
      mbar_wait(bars + 1, ph_k);  // the group's K^ row has landed
      ph_k ^= 1;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = cmul(v[e], kb[fold_index(in_pos<RL, LANES, 0>(lane, e), L)]);
    sync();  // K^ row consumed
    prefetch_k(line + stride);
    int ky, kx;
    coords(line, ky, kx);
    RowOut dst{a.out + ky * a.out_si + int64_t(kx) * a.out_sk, 1, a.out_nvalid, true, a.scale};
    warp_fft<RL, LANES, true, kPout>(v, ex, lane, tw, vin, dst, sync);
  }
  if constexpr (!BULK) cp_async_wait0();
}

// Transposing passes on multi-warp lines (L = 1024..2048, where a one-warp line spills and an
// 8-line [pos][8] tile no longer fits): persistent CTAs of T lines x LANES lanes.  Each line has
// a private swizzled exchange buffer X (stride L + 8/T: the skew makes the cooperative tile
// reads / stores below bank-conflict-free); stages synchronise the line's warps with a named
// barrier.
//   mw_row_to_col (A, B): every line group stages its own next input row by cp.async while the
//     current one is transformed; the last stage lands in X and, after one CTA barrier, the CTA
//     stores position-major segments of T adjacent lines (T x 16 B contiguous).
//   mw_col_to_row (D, E): the CTA stages the next [pos][T] column tile (swizzled) by cp.async
//     while each group transforms its column of the current one and stores its output row from
//     registers.
// the line's exchange barrier: __syncwarp for one-warp lines, a named barrier (id 1 + group)
// over the group's warps otherwise
template <int LANES>
struct LineSync {
  using type = GroupSync<LANES>;
  static __device__ __forceinline__ type make(int grp) { return type{1 + grp}; }
};
template <>
struct LineSync<32> {
  using type = WarpSync;
  static __device__ __forceinline__ type make(int) { return type{}; }
};


template <int L, int T>
struct MWSmem {
  static constexpr int XSTRIDE = L + 8 / T;
  static constexpr size_t R2C_BYTES = (size_t(T) * XSTRIDE + size_t(T) * (L / 2)) * sizeof(double2);
  static constexpr size_t C2R_BYTES = (size_t(T) * XSTRIDE + size_t(T) * L) * sizeof(double2);
};

template <class RL, int LANES, int T, int MINB>
__global__ void __launch_bounds__(T * LANES, MINB) mw_row_to_col(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int R0 = RL::at(0);
  using SM = MWSmem<L, T>;
  static_assert(T == 2 || T == 4 || T == 8, "tile lines");
  extern __shared__ double2 sm[];
  const int grp = threadIdx.x / LANES, lane = threadIdx.x % LANES;
  const typename LineSync<LANES>::type sync = LineSync<LANES>::make(grp);
  double2* const xb = sm + grp * SM::XSTRIDE;
  double2* const sb = sm + T * SM::XSTRIDE + grp * (L / 2);  // staged input row (pruned: < L/2)
  const int ntiles_i = (a.n_inner + T - 1) / T;
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto prefetch = [&](int64_t tix) {
    if (tix < ntiles) {
      const int i = int(unsigned(tix) % unsigned(ntiles_i)) * T + grp;
      const int k = int(unsigned(tix) / unsigned(ntiles_i));
      if (i < a.n_inner) {
        const double2* in = a.in + int64_t(i) * a.in_si + int64_t(k) * a.in_sk;
        for (int pos = lane; pos < a.in_nvalid; pos += LANES) cp_async16(sb + swz(pos), in + pos);
      }
    }
    cp_async_commit();
  };
  const TwTable tw{a.tw};
  const PrivEx ex{xb};
  int64_t tix = blockIdx.x;
  prefetch(tix);
  for (; tix < ntiles; tix += gridDim.x) {
    const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
    const int k = int(unsigned(tix) / unsigned(ntiles_i));
    const int lines_ok = min(T, a.n_inner - i0);
    cp_async_wait0();
    sync();  // the group's own staged row has landed
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (R0 == 8 && (e % R0) >= R0 / 2) continue;  // zero padding: not staged
      const int pos = in_pos<RL, LANES, 0>(lane, e);
      v[e] = pos < a.in_nvalid ? sb[swz(pos)] : make_double2(0.0, 0.0);
    }
    sync();  // staging consumed by the group: refill it with the next tile's row
    prefetch(tix + gridDim.x);
    RegsIn vin{v};
    RegsOut vout{v};
    warp_fft<RL, LANES, false, 1>(v, ex, lane, tw, vin, vout, sync);
    sync();  // every lane of the group is done reading X (last exchange)
#pragma unroll
    for (int e = 0; e < E; ++e) ex.at(out_pos<RL, LANES, RL::n - 1>(lane, e)) = v[e];
    __syncthreads();  // all T lines are in X
    double2* const base = a.out + int64_t(i0) * a.out_si + int64_t(k) * a.out_sk;
    for (int e = threadIdx.x; e < a.out_nvalid * T; e += T * LANES) {
      const int pos = e / T, t = e % T;
      if (t < lines_ok) {
        const double2 x = sm[t * SM::XSTRIDE + swz(pos)];
        const double2 y = (a.scale == 1.0) ? x : cscale(x, a.scale);
        if (a.pm.n == 0) {
          base[t * a.out_si + pos * a.out_sp] = y;
        } else {  // fused transpose: the segment goes straight to the rank owning it
          const int q = a.pm.owner(a.pm.by_pos ? pos : i0 + t);
          a.pm.base[q][a.pm.off[q] + int64_t(i0 + t) * a.out_si + int64_t(k) * a.pm.sk[q] + int64_t(pos) * a.out_sp] = y;
        }
      }
    }
    __syncthreads();  // X read out before the next tile's first exchange
  }
  cp_async_wait0();
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

template <class RL, int LANES, int T, int MINB>
__global__ void __launch_bounds__(T * LANES, MINB) mw_col_to_row(WArgs a) {
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  using SM = MWSmem<L, T>;
  static_assert(T == 2 || T == 4 || T == 8, "tile lines");
  extern __shared__ double2 sm[];
  const int grp = threadIdx.x / LANES, lane = threadIdx.x % LANES;
  const typename LineSync<LANES>::type sync = LineSync<LANES>::make(grp);
  double2* const tile = sm + T * SM::XSTRIDE;
  const int ntiles_i = (a.n_inner + T - 1) / T;
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto prefetch = [&](int64_t tix) {
    if (tix < ntiles) {
      const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
      const int k = int(unsigned(tix) / unsigned(ntiles_i));
      const int lines_ok = min(T, a.n_inner - i0);
      const double2* base = a.in + int64_t(i0) * a.in_si + int64_t(k) * a.in_sk;
      for (int e = threadIdx.x; e < a.in_nvalid * T; e += T * LANES) {
        const int pos = e / T, t = e % T;
        cp_async16_zfill(&tile[mtile_at<T>(pos, t)], t < lines_ok ? base + t * a.in_si + pos * a.in_sp : a.in,
                         t < lines_ok);
      }
    }
    cp_async_commit();
  };
  const TwTable tw{a.tw};
  const PrivEx ex{sm + grp * SM::XSTRIDE};
  int64_t tix = blockIdx.x;
  prefetch(tix);
  for (; tix < ntiles; tix += gridDim.x) {
    const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
    const int k = int(unsigned(tix) / unsigned(ntiles_i));
    const bool ok = grp < min(T, a.n_inner - i0);
    cp_async_wait0();
    __syncthreads();  // this tile's copies (issued by all threads) have landed
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int pos = in_pos<RL, LANES, 0>(lane, e);
      v[e] = pos < a.in_nvalid ? tile[mtile_at<T>(pos, grp)] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // tile consumed by every group
    prefetch(tix + gridDim.x);
    const int line = i0 + (ok ? grp : 0);
    RegsIn vin{v};
    double2* orow = a.out + int64_t(line) * a.out_si + int64_t(k) * a.out_sk;
    if (a.pm.n) {  // fused transpose: the row goes straight to the rank owning line (z)
      const int q = a.pm.owner(line);
      orow = a.pm.base[q] + (a.pm.off[q] + int64_t(line) * a.out_si + int64_t(k) * a.pm.sk[q]);
    }
    RowOut dst{orow, 1, a.out_nvalid, ok, a.scale};
    warp_fft<RL, LANES, true, 2>(v, ex, lane, tw, vin, dst, sync);  // cropped output half
  }
  cp_async_wait0();
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

// FUSG_PP_WAVES: CTAs per resident slot of the persistent warp kernels of the other lengths
// (pass C, multi-warp lines, D/E col->row); 1 = fully persistent.  8: 768^3 apply 73.5 -> 71.8
// ms, 323^3 6.17 -> 6.12 ms (the block scheduler's relaunches desynchronise the warps).
static int pp_waves() {
  static const int w = [] {
    const char* e = getenv("FUSG_PP_WAVES");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  return w;
}

struct MWVariant {
  int L;
  bool r2c, def;
  int lanes, T;
  WFn fn;
  size_t smem;
};
#define FUSG_MW_R2C(DEF, LANES, T, MINB, ...)                                               \
  MWVariant {                                                                               \
    Radices<__VA_ARGS__>::len(), true, DEF, LANES, T, mw_row_to_col<Radices<__VA_ARGS__>, LANES, T, MINB>, \
        MWSmem<Radices<__VA_ARGS__>::len(), T>::R2C_BYTES                                   \
  }
#define FUSG_MW_C2R(DEF, LANES, T, MINB, ...)                                               \
  MWVariant {                                                                               \
    Radices<__VA_ARGS__>::len(), false, DEF, LANES, T, mw_col_to_row<Radices<__VA_ARGS__>, LANES, T, MINB>, \
        MWSmem<Radices<__VA_ARGS__>::len(), T>::C2R_BYTES                                   \
  }
// Variants per (length, direction); FUSG_MW_<L>_R2C / _C2R = index among them (-1: static
// kernels), else the one marked default.  Measured (tools/pass_times.py, ms for A B D E):
//   1536 (768^3): static 8.8 17.4 17.8 8.5 -> 6.7 12.7 11.0 6.3 (apply 86.1 -> 70.4 ms);
//                 T = 2 tiles: 12.5 14.0 10.8 11.6; 128-lane lines (12 points per lane, radices
//                 4,4,4,4,2,3, 16 warps per SM): 8.8 17.4 17.9 8.6 (pass C 4,4,2,3,4,4: 63 vs 34 ms)
//   1024 (512^3): static 1.95 3.75 3.93 2.03 -> r2c 1.96 3.76 (kept static), c2r 3.33 1.88
//   512 (cfg2): pp warp kernels 0.156 0.297 0.344 0.178 -> c2r on 4-line tiles (3 CTAs, 12
//                 warps per SM) 0.295 0.166 (apply 1.861 -> 1.800 ms); 8-line tiles 0.348 0.180;
//                 4 CTAs at 128 registers 0.301 0.172; 2-line tiles 0.349+; r2c 0.18 0.34 (kept warp)
//   2048 (1024^3): static 19.5 38.5 38.7 19.6 -> 29.6 52.0 34.8 29.6 with T = 2 (32-byte
//                 segments at a 16 MB position stride in pass E): kept static
static const MWVariant kMW[] = {
    FUSG_MW_R2C(true, 64, 4, 1, 8, 8, 3, 8),  // 1536: 24 points per lane
    FUSG_MW_R2C(false, 64, 2, 2, 8, 8, 3, 8),
    FUSG_MW_C2R(true, 64, 4, 1, 8, 8, 3, 8),
    FUSG_MW_C2R(false, 64, 2, 1, 8, 8, 3, 8),
    FUSG_MW_R2C(false, 64, 4, 1, 8, 4, 4, 8),  // 1024: 16 points per lane
    FUSG_MW_R2C(false, 128, 4, 1, 8, 4, 4, 8),
    FUSG_MW_C2R(true, 64, 4, 1, 8, 4, 4, 8),
    FUSG_MW_C2R(false, 128, 4, 1, 8, 4, 4, 8),
    FUSG_MW_R2C(false, 32, 4, 3, 8, 8, 8),  // 512: one-warp lines, 4- / 8-line tiles
    FUSG_MW_R2C(false, 32, 8, 1, 8, 8, 8),
    FUSG_MW_C2R(true, 32, 4, 3, 8, 8, 8),
    FUSG_MW_C2R(false, 32, 8, 1, 8, 8, 8),
    FUSG_MW_R2C(false, 128, 2, 1, 8, 4, 8, 8),  // 2048: 16 points per lane
    FUSG_MW_C2R(false, 128, 2, 1, 8, 4, 8, 8),
};
#undef FUSG_MW_R2C
#undef FUSG_MW_C2R

// Transposing pass on multi-warp lines: 1 launched, 0 not applicable, -1 error.  Pruned halves
// only (zero-padded input of row_to_col, cropped output of col_to_row), as in every apply.
static int launch_mw(fusg_ctx* ctx, int L, bool r2c, const WArgs& a, cudaStream_t s) {
  if (r2c ? 2 * a.in_nvalid > L : 2 * a.out_nvalid > L) return 0;
  const std::string var_name = "FUSG_MW_" + std::to_string(L) + (r2c ? "_R2C" : "_C2R");
  const char* ve = getenv(var_name.c_str());
  const int want = ve ? atoi(ve) : -2;
  if (want == -1) return 0;
  const MWVariant* v = nullptr;
  const MWVariant* first = nullptr;
  int seen = 0;
  for (const auto& c : kMW)
    if (c.L == L && c.r2c == r2c) {
      if (!first) first = &c;
      if (want >= 0 ? seen == want : c.def) {
        v = &c;
        break;
      }
      ++seen;
    }
  if (!v && a.pm.n && want < 0) v = first;  // fused peer stores need a transposing kernel
  if (!v) return 0;
  if (cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(v->smem)) != cudaSuccess) {
    set_error(FUSG_CUDA, "multi-warp transposing pass: cannot configure shared memory");
    return -1;
  }
  const int threads = v->T * v->lanes;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v->fn, threads, v->smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  const int64_t tiles = int64_t((a.n_inner + v->T - 1) / v->T) * a.n_outer;
  const int64_t grid = std::min<int64_t>(tiles, int64_t(per_sm) * ctx->num_sms * pp_waves());
  v->fn<<<unsigned(grid), threads, v->smem, s>>>(a);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "multi-warp transposing pass");
    return -1;
  }
  return 1;
}


// FUSG_BULK=0: pass C stages its rows with per-lane cp.async instead of 1-D bulk copies
static int bulk_staging() {
  static const int on = [] {
    const char* e = getenv("FUSG_BULK");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

struct PPMVariant {
  int L, lanes, groups;
  WFn fn[2];  // [bulk staging]
  size_t smem;
};
#define FUSG_PPM(LANES, GROUPS, MINB, ...)                                                  \
  PPMVariant {                                                                              \
    Radices<__VA_ARGS__>::len(), LANES, GROUPS,                                             \
        {warp_row_conv_pp64<Radices<__VA_ARGS__>, LANES, GROUPS, MINB, true, false>,         \
         warp_row_conv_pp64<Radices<__VA_ARGS__>, LANES, GROUPS, MINB, true, true>},         \
        PP64Smem<Radices<__VA_ARGS__>::len(), true, GROUPS>::BYTES                          \
  }
// Variants per length, selected by FUSG_PPM_<L> (index; -1 = none: 512/1024 then run the
// one-warp pp kernel).  The first entry of each length is the default.
static const PPMVariant kPPM[] = {
    FUSG_PPM(64, 2, 1, 8, 8, 3, 8),   // 1536: 24 points per lane
    FUSG_PPM(128, 1, 3, 8, 4, 8, 8),  // 2048: 16 per lane (64 lanes: 118 ms at 1024^3; 256: 93; this: 81)
    FUSG_PPM(64, 1, 6, 8, 4, 4, 8),   // 1024: 16 per lane (one warp: 14.4 ms at 512^3; 128 lanes: 10.6; this: 9.4)
    // 512 and 768 stay on one-warp lines: 64-lane variants measured 1.05-1.08 ms against 0.89
    // (cfg2 pass C) and 5.7 ms against 4.0 (384^3, 12 points per lane on radices 4,4,3,4,4)
};
#undef FUSG_PPM

// the multi-warp-line persistent pass C, or 0 when not applicable
static int launch_conv64(fusg_ctx* ctx, int L, const WArgs& a, cudaStream_t s) {
  static const bool on = [] {
    const char* e = getenv("FUSG_CONV_PP64");
    return !(e && atoi(e) == 0);
  }();
  if (!on || 2 * a.in_nvalid > L || 2 * a.out_nvalid > L || a.in_nvalid < 1) return 0;  // pruned halves only
  const std::string var_name = "FUSG_PPM_" + std::to_string(L);
  const char* ve = getenv(var_name.c_str());
  const int def = 0;
  const int want = ve ? atoi(ve) : def;
  if (want < 0) return 0;
  const PPMVariant* v = nullptr;
  int seen = 0;
  for (const auto& c : kPPM)
    if (c.L == L && seen++ == want) v = &c;
  if (!v) return 0;
  const WFn fn = v->fn[bulk_staging()];
  const size_t smem = v->smem;
  const int groups = v->groups, lanes = v->lanes;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
    set_error(FUSG_CUDA, "long-line pass C: cannot configure shared memory");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, groups * lanes, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  const int64_t lines = int64_t(a.n_inner) * a.n_outer;
  const int64_t grid = std::min<int64_t>((lines + groups - 1) / groups, int64_t(per_sm) * ctx->num_sms * pp_waves());
  fn<<<unsigned(grid), groups * lanes, smem, s>>>(a);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "long-line pass C");
    return -1;
  }
  return 1;
}

template <class RL, int LN, bool PRUNED>
constexpr WFn colrow_pp_ptr() {
  if constexpr (LN == 32 && whole_butterflies<RL>(32)) return warp_col_to_row_pp<RL, PRUNED>;
  else return nullptr;
}
template <class RL, int LN, bool PRUNED, bool BULK>
constexpr WFn conv_pp_ptr() {
  if constexpr (LN == 32 && whole_butterflies<RL>(32)) return warp_row_conv_pp<RL, 32, PRUNED, BULK>;
  else return nullptr;
}

template <class RL, int LN, bool INV, bool PRUNED>
constexpr WFn transpose_ptr() {
  if constexpr (LN == 32 && whole_butterflies<RL>(32)) {
    if constexpr (INV) return warp_col_to_row<RL, true, PRUNED>;
    else return warp_row_to_col<RL, false, PRUNED>;
  } else {
    return nullptr;
  }
}

struct WarpEntry {
  int L, lanes;
  WFn fwd, inv, conv;
  WFn row_to_col_fwd[2], col_to_row_inv[2];  // transposing passes (LANES = 32), [pruned]
  WFn conv_pp[2][2];  // persistent pipelined pass C, [pruned][bulk staging] (nullptr: not available)
  size_t pp_smem[2];
  WFn col_to_row_pp[2];  // persistent pipelined inverse column -> row (passes D, E), [pruned]
};
#define FUSG_WARP(LN, ...)                                                                  \
  WarpEntry {                                                                               \
    Radices<__VA_ARGS__>::len(), LN, warp_line_pass<Radices<__VA_ARGS__>, LN, false>,       \
        warp_line_pass<Radices<__VA_ARGS__>, LN, true>, warp_row_conv<Radices<__VA_ARGS__>, LN>, \
        {transpose_ptr<Radices<__VA_ARGS__>, LN, false, false>(),                              \
         transpose_ptr<Radices<__VA_ARGS__>, LN, false, true>()},                              \
        {transpose_ptr<Radices<__VA_ARGS__>, LN, true, false>(),                               \
         transpose_ptr<Radices<__VA_ARGS__>, LN, true, true>()},                               \
        {{conv_pp_ptr<Radices<__VA_ARGS__>, LN, false, false>(), conv_pp_ptr<Radices<__VA_ARGS__>, LN, false, true>()}, \
         {conv_pp_ptr<Radices<__VA_ARGS__>, LN, true, false>(), conv_pp_ptr<Radices<__VA_ARGS__>, LN, true, true>()}}, \
        {PPConvSmem<Radices<__VA_ARGS__>::len(), false>::BYTES,                                  \
         PPConvSmem<Radices<__VA_ARGS__>::len(), true>::BYTES},                                  \
        {colrow_pp_ptr<Radices<__VA_ARGS__>, LN, false>(), colrow_pp_ptr<Radices<__VA_ARGS__>, LN, true>()} \
  }
// pass-C-only entry: the persistent pass C alone (the row/column kernels would spill at this E)
#define FUSG_WARP_CONV_ONLY(LN, ...)                                                         \
  WarpEntry {                                                                               \
    Radices<__VA_ARGS__>::len(), LN, nullptr, nullptr, nullptr, {nullptr, nullptr}, {nullptr, nullptr}, \
        {{conv_pp_ptr<Radices<__VA_ARGS__>, LN, false, false>(), conv_pp_ptr<Radices<__VA_ARGS__>, LN, false, true>()}, \
         {conv_pp_ptr<Radices<__VA_ARGS__>, LN, true, false>(), conv_pp_ptr<Radices<__VA_ARGS__>, LN, true, true>()}}, \
        {PPConvSmem<Radices<__VA_ARGS__>::len(), false>::BYTES,                                  \
         PPConvSmem<Radices<__VA_ARGS__>::len(), true>::BYTES},                                  \
        {nullptr, nullptr}                                                                       \
  }
static const WarpEntry kWarpTab[] = {
    FUSG_WARP(32, 8, 8, 8),  // 512 (cfg2)
    FUSG_WARP(32, 8, 4, 3, 8),  // 768 (pass C for Nz <= 384: the nested cascade grids)
    FUSG_WARP_CONV_ONLY(32, 8, 4, 4, 8),  // 1024 (pass C for Nz <= 512: cfg3)
    FUSG_WARP(32, 8, 4, 8),  // 256
    FUSG_WARP(16, 8, 2, 8),  // 128 (cfg1)
};

enum WarpMode { kWRow = 0, kWCol = 1, kWConv = 2, kWRowToCol = 3, kWColToRow = 4 };

// FUSG_WARP=0 disables the warp engine.  Returns 1 launched, 0 not applicable, -1 error.
static int launch_warp(fusg_ctx* ctx, int L, int mode, bool inv, const WArgs& a, cudaStream_t s) {
  static const bool enabled = [] {
    const char* e = getenv("FUSG_WARP");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled) return 0;
  const WarpEntry* we = nullptr;
  for (const auto& e : kWarpTab)
    if (e.L == L) we = &e;
  if (!we) return 0;
  static const int disable_mask = [] {  // FUSG_WARP_OFF bitmask: 1 rows, 2 columns, 4 conv
    const char* e = getenv("FUSG_WARP_OFF");
    return e ? atoi(e) : 0;
  }();
  if (disable_mask & (1 << mode)) return 0;
  WFn fn = mode == kWConv ? we->conv : (inv ? we->inv : we->fwd);
  if (mode == kWConv && inv) return 0;
  if (!we->fwd && mode != kWConv) return 0;  // pass-C-only entry
  if (mode == kWRowToCol || mode == kWColToRow) {
    // pruned radix-8 end stages when the zero padding / crop covers the upper half
    const bool pr = mode == kWRowToCol ? 2 * a.in_nvalid <= L : 2 * a.out_nvalid <= L;
    static const bool colrow_pp = [] {  // FUSG_COLROW_PP=0: one tile per CTA, no pipelining
      const char* e = getenv("FUSG_COLROW_PP");
      return !(e && atoi(e) == 0);
    }();
    if (a.pm.n && mode == kWColToRow && !we->col_to_row_pp[pr]) return 0;  // fused stores: pp kernel only
    if (mode == kWColToRow && inv && (colrow_pp || a.pm.n) && we->col_to_row_pp[pr]) {
      WFn pp = we->col_to_row_pp[pr];
      const size_t psmem = size_t(L) * 8 * 2 * sizeof(double2);  // two tile buffers
      if (cudaFuncSetAttribute(pp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(psmem)) != cudaSuccess) {
        set_error(FUSG_CUDA, "persistent column->row pass: cannot configure shared memory");
        return -1;
      }
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pp, kWarpThreads, psmem) == cudaSuccess &&
          per_sm >= 1) {
        const int64_t tiles = int64_t((a.n_inner + 7) / 8) * a.n_outer;
        const int64_t grid = std::min<int64_t>(tiles, int64_t(per_sm) * ctx->num_sms * pp_waves());
        pp<<<unsigned(grid), kWarpThreads, psmem, s>>>(a);
        ctx->launches++;
        const cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
          cuda_error(err, "persistent column->row pass");
          return -1;
        }
        return 1;
      }
      cudaGetLastError();
    }
    fn = mode == kWRowToCol ? (inv ? nullptr : we->row_to_col_fwd[pr]) : (inv ? we->col_to_row_inv[pr] : nullptr);
    if (!fn) return 0;
    const size_t tsmem = size_t(L) * 8 * sizeof(double2);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsmem)) != cudaSuccess) {
      set_error(FUSG_CUDA, "transposing warp pass: cannot configure shared memory");
      return -1;
    }
    const int64_t tb = int64_t((a.n_inner + 7) / 8) * a.n_outer;
    fn<<<unsigned(tb), kWarpThreads, tsmem, s>>>(a);
    ctx->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
      cuda_error(err, "transposing warp pass");
      return -1;
    }
    return 1;
  }
  static const bool use_pp = [] {  // FUSG_CONV_PP=0 selects the one-line-per-warp pass C
    const char* e = getenv("FUSG_CONV_PP");
    return !(e && atoi(e) == 0);
  }();
  const int pruned = 2 * a.in_nvalid <= L && 2 * a.out_nvalid <= L;
  const WFn conv_pp = a.in_nvalid >= 1 ? we->conv_pp[pruned][bulk_staging()] : nullptr;
  const size_t pp_smem = we->pp_smem[pruned];
  if (mode == kWConv && use_pp && L == 512 && bulk_staging()) {  // 16 x 16 x 2 pass C (conv_r16.cu)
    const int r = launch_conv_r16(ctx, a, s);
    if (r != 0) return r;
  }
  if (mode == kWConv && use_pp && conv_pp) {
    if (cudaFuncSetAttribute(conv_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pp_smem)) != cudaSuccess) {
      set_error(FUSG_CUDA, "persistent pass C: cannot configure shared memory");
      return -1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_pp, kPPWarps * 32, pp_smem) !=
            cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      return 0;
    }
    const int64_t lines = int64_t(a.n_inner) * a.n_outer;
    const int64_t grid = std::min<int64_t>((lines + kPPWarps - 1) / kPPWarps, int64_t(per_sm) * ctx->num_sms * pp_waves());
    conv_pp<<<unsigned(grid), kPPWarps * 32, pp_smem, s>>>(a);
    ctx->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
      cuda_error(err, "persistent pass C");
      return -1;
    }
    return 1;
  }
  if (!fn) return 0;  // pass-C-only entry without an applicable persistent variant
  const int lpc = kWarpThreads / we->lanes;
  const size_t smem = size_t(lpc) * L * sizeof(double2);
  const int64_t blocks = (int64_t(a.n_inner) * a.n_outer + lpc - 1) / lpc;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
    set_error(FUSG_CUDA, "warp pass: cannot configure shared memory");
    return -1;
  }
  fn<<<unsigned(blocks), kWarpThreads, smem, s>>>(a);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "warp fft pass");
    return -1;
  }
  return 1;
}

template <class Fn, class... Args>
static fusg_status launch_static(fusg_ctx* ctx, Fn fn, const StaticEntry& e, int n_inner, int n_outer,
                                 cudaStream_t s, Args... args) {
  LineGeom g{n_inner, n_outer, (n_inner + e.T - 1) / e.T};
  const size_t smem = size_t(e.L) * (e.T + 1) * sizeof(double2);  // tile + twiddles
  FUSG_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t blocks = int64_t(g.ntiles) * n_outer;
  fn<<<unsigned(blocks), e.threads, smem, s>>>(g, args...);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("static fft pass");
  return FUSG_OK;
}

template <bool INV, int T, class LD, class ST>
static fusg_status launch_axis_t(fusg_ctx* ctx, const AxisPlan& pl, int n_inner, int n_outer,
                                 const LD& ld, const ST& st, cudaStream_t s) {
  LineGeom g{n_inner, n_outer, (n_inner + T - 1) / T};
  const size_t smem = size_t(pl.L) * T * sizeof(double2);
  auto fn = axis_pass<INV, T, LD, ST>;
  FUSG_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t blocks = int64_t(g.ntiles) * n_outer;
  fn<<<unsigned(blocks), T * pl.tpl, smem, s>>>(pl, g, ld, st);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("axis_pass");
  return FUSG_OK;
}

template <bool INV, class LD, class ST>
static fusg_status launch_axis(fusg_ctx* ctx, const AxisPlan& pl, int n_inner, int n_outer,
                               const LD& ld, const ST& st, cudaStream_t s, int kind = kKindCol) {
  if (size_t(pl.L) * sizeof(double2) > 200 * 1024)
    return set_error(FUSG_INVALID_ARGUMENT, "padded axis length too large for one CTA");
  if constexpr (std::is_same<LD, GLoadF>::value && std::is_same<ST, GStoreF>::value) {
    const bool rows = kind == kKindRow;
    // FUSG_WARP_TRANSPOSE bitmask: 1 row->col (forward A, B; default), 2 col->row (inverse D, E;
    // measured slower than the row-staged CTA kernels: its cooperative load couples the warps)
    static const int wt = [] {
      const char* v = getenv("FUSG_WARP_TRANSPOSE");
      return v ? atoi(v) : 1;
    }();
    const bool r2c = !INV && ld.g.sp == 1 && st.g.si == 1 && st.g.sp != 1 && (wt & 1);
    static const bool colrow_pp = [] {
      const char* v = getenv("FUSG_COLROW_PP");
      return !(v && atoi(v) == 0);
    }();
    const bool c2r = INV && ld.g.si == 1 && ld.g.sp != 1 && st.g.sp == 1 && ((wt & 2) || colrow_pp);
    if (r2c || c2r) {
      const WArgs wa{ld.g.p, ld.g.si, ld.g.sk, ld.g.sp, ld.g.nvalid, st.g.p, st.g.si, st.g.sk,
                     st.g.sp, st.g.nvalid, st.g.scale, n_inner, n_outer, pl.tw, KOct{}};
      int r = pl.L == 512 ? launch_transpose_r16(ctx, r2c, wa, s)
              : pl.L == 1536 ? launch_transpose_r16x3(ctx, r2c, wa, s)
              : pl.L == 1024 ? launch_transpose_r16x2(ctx, r2c, wa, s) : 0;
      if (r == 0) r = launch_mw(ctx, pl.L, r2c, wa, s);
      if (r == 0) r = launch_warp(ctx, pl.L, r2c ? kWRowToCol : kWColToRow, INV, wa, s);
      if (r < 0) return FUSG_CUDA;
      if (r > 0) return FUSG_OK;
    }
    if ((rows && ld.g.sp == 1 && st.g.sp == 1) || (!rows && ld.g.si == 1 && st.g.si == 1)) {
      const WArgs wa{ld.g.p, ld.g.si, ld.g.sk, ld.g.sp, ld.g.nvalid, st.g.p, st.g.si, st.g.sk,
                     st.g.sp, st.g.nvalid, st.g.scale, n_inner, n_outer, pl.tw, KOct{}};
      const int r = launch_warp(ctx, pl.L, rows ? kWRow : kWCol, INV, wa, s);
      if (r < 0) return FUSG_CUDA;
      if (r > 0) return FUSG_OK;
    }
    if (const StaticEntry* e = find_static(pl.L, kind)) {
      // FUSG_STAGE_ROWS bitmask: 1 stage row loads (measured neutral), 2 stage row stores
      static const int stage_rows = [] {
        const char* v = getenv("FUSG_STAGE_ROWS");
        return v ? atoi(v) : 2;
      }();
      AxisFn fn = INV ? e->inv : e->fwd;
      if ((stage_rows & 1) && !INV && ld.g.sp == 1 && st.g.sp != 1) fn = e->fwd_rowin;
      if ((stage_rows & 2) && INV && st.g.sp == 1 && ld.g.sp != 1) fn = e->inv_rowout;
      return launch_static(ctx, fn, *e, n_inner, n_outer, s, ld, st, pl.tw);
    }
  }
  // kernel-spectrum build passes (generate / fold + forward) on compile-time plans
  if constexpr (!INV && std::is_same<ST, GStoreF>::value &&
                (std::is_same<LD, KGenF>::value || std::is_same<LD, FoldF>::value)) {
    if (const StaticEntry* e = find_static(pl.L, kKindCol)) {
      if constexpr (std::is_same<LD, KGenF>::value) {
        if (e->build_gen) return launch_static(ctx, e->build_gen, *e, n_inner, n_outer, s, ld, st, pl.tw);
      } else {
        if (e->build_fold) return launch_static(ctx, e->build_fold, *e, n_inner, n_outer, s, ld, st, pl.tw);
      }
    }
  }
  switch (choose_tile(pl, n_inner)) {
    case 16: return launch_axis_t<INV, 16>(ctx, pl, n_inner, n_outer, ld, st, s);
    case 8: return launch_axis_t<INV, 8>(ctx, pl, n_inner, n_outer, ld, st, s);
    case 4: return launch_axis_t<INV, 4>(ctx, pl, n_inner, n_outer, ld, st, s);
    case 2: return launch_axis_t<INV, 2>(ctx, pl, n_inner, n_outer, ld, st, s);
    default: return launch_axis_t<INV, 1>(ctx, pl, n_inner, n_outer, ld, st, s);
  }
}

template <int T>
static fusg_status launch_conv_t(fusg_ctx* ctx, const AxisPlan& pl, int n_inner, int n_outer,
                                 const GLoadF& ld, const GStoreF& st, const KOct& ko,
                                 cudaStream_t s) {
  LineGeom g{n_inner, n_outer, (n_inner + T - 1) / T};
  const size_t smem = size_t(pl.L) * T * sizeof(double2);
  auto fn = conv_pass<T>;
  FUSG_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t blocks = int64_t(g.ntiles) * n_outer;
  const int fuse = pl.radix[0] == pl.radix[pl.nst - 1];
  fn<<<unsigned(blocks), T * pl.tpl, smem, s>>>(pl, g, ld, st, ko, fuse);
  ctx->launches++;
  FUSG_LAUNCH_CHECK("conv_pass");
  return FUSG_OK;
}

static fusg_status launch_conv(fusg_ctx* ctx, const AxisPlan& pl, int n_inner, int n_outer,
                               const GLoadF& ld, const GStoreF& st, const KOct& ko,
                               cudaStream_t s) {
  if (size_t(pl.L) * sizeof(double2) > 200 * 1024)
    return set_error(FUSG_INVALID_ARGUMENT, "padded axis length too large for one CTA");
  if (ld.g.sp == 1 && st.g.sp == 1 && ko.s_kz == 1) {
    const WArgs wa{ld.g.p, ld.g.si, ld.g.sk, ld.g.sp, ld.g.nvalid, st.g.p, st.g.si, st.g.sk,
                   st.g.sp, st.g.nvalid, st.g.scale, n_inner, n_outer, pl.tw, ko};
    int r = pl.L == 1536 ? launch_conv_r16x3(ctx, wa, s)
            : pl.L == 1024 ? launch_conv_r16x2(ctx, wa, s)
            : pl.L == 768 ? launch_conv_r16x3h(ctx, wa, s) : 0;
    if (r == 0) r = launch_conv64(ctx, pl.L, wa, s);
    if (r == 0) r = launch_warp(ctx, pl.L, kWConv, false, wa, s);
    if (r < 0) return FUSG_CUDA;
    if (r > 0) return FUSG_OK;
  }
  if (const StaticEntry* e = find_static(pl.L, kKindConv))
    return launch_static(ctx, e->conv, *e, n_inner, n_outer, s, ld, st, ko, pl.tw);
  switch (choose_tile(pl, n_inner)) {
    case 16: return launch_conv_t<16>(ctx, pl, n_inner, n_outer, ld, st, ko, s);
    case 8: return launch_conv_t<8>(ctx, pl, n_inner, n_outer, ld, st, ko, s);
    case 4: return launch_conv_t<4>(ctx, pl, n_inner, n_outer, ld, st, ko, s);
    case 2: return launch_conv_t<2>(ctx, pl, n_inner, n_outer, ld, st, ko, s);
    default: return launch_conv_t<1>(ctx, pl, n_inner, n_outer, ld, st, ko, s);
  }
}

// ---------------------------------------------------------------------------- build
void slab_split(int n, int G, int r, int* begin, int* count) {
  const int base = n / G, extra = n % G;  // the first `extra` ranks take one more (ragged)
  *count = base + (r < extra ? 1 : 0);
  *begin = r * base + std::min(r, extra);
}

fusg_status kernel_init_geometry(fusg_kernel* K, int G, int rank) {
  for (int a = 0; a < 3; ++a) {
    K->P[a] = device_padded_size(K->grid.dims[a], a);
    K->H[a] = K->P[a] / 2 + 1;
    if (!make_plan_radices(K->P[a], K->plan[a]))
      return set_error(FUSG_INVALID_ARGUMENT, "no FFT plan for padded length");
  }
  if (G < 1 || rank < 0 || rank >= G) return set_error(FUSG_INVALID_ARGUMENT, "bad slab rank");
  if (G > K->grid.dims[2] || G > K->P[0])
    return set_error(FUSG_INVALID_ARGUMENT, "more ranks than z-planes or kx columns");
  K->G = G;
  K->rank = rank;
  K->zs.resize(G);
  K->nzs.resize(G);
  K->xs.resize(G);
  K->nxs.resize(G);
  for (int r = 0; r < G; ++r) {
    slab_split(K->grid.dims[2], G, r, &K->zs[r], &K->nzs[r]);
    slab_split(K->P[0], G, r, &K->xs[r], &K->nxs[r]);
  }
  K->z0 = K->zs[rank];
  K->nz = K->nzs[rank];
  K->x0 = K->xs[rank];
  K->nx = K->nxs[rank];
  // Unsharded kernels keep A as [z][kx][y]: passes A and E then move their 64/128-byte kx
  // segments at an Ny-element stride instead of Nz*Ny, staying within DRAM pages (cfg5: A 6.25
  // -> 5.22 ms, E 6.30 -> 5.45 ms; cfg2 neutral).  FUSG_A_ZKY=0 restores [kx][z][y], the
  // layout of the sharded kernels' x-slabs.
  static const bool zky = [] {
    const char* e = getenv("FUSG_A_ZKY");
    return !(e && atoi(e) == 0);
  }();
  // B's z pitch: with Nz = 487 (cfg3) the 64-byte tile segments of passes B and D straddled
  // 128-byte lines (pass B at 0.48 of HBM against 0.78 at Nz = 512)
  static const bool bpitch = [] {
    const char* e = getenv("FUSG_B_PITCH");
    return !(e && atoi(e) == 0);
  }();
  const int64_t Nz = K->grid.dims[2];
  K->bz = bpitch ? (Nz + 7) / 8 * 8 : Nz;
  const int64_t Ny = K->grid.dims[1];
  if (zky && G == 1 && !K->slab) {
    K->az = int64_t(K->P[0]) * Ny;
    K->akx = Ny;
  } else {
    K->az = Ny;
    K->akx = int64_t(K->nz) * Ny;  // x-slab X and the A slab: [kx][z in slab][y]
  }
  return FUSG_OK;
}

fusg_status volume_potential_build(fusg_kernel* K, double2 self) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  for (int a = 0; a < 3; ++a) {
    FUSG_TRY(upload_twiddles(K->ctx, K->P[a], &K->tw[a]));
    K->plan[a].tw = K->tw[a];
  }
  const int Px = K->P[0], Py = K->P[1], Pz = K->P[2];
  const int Hx = K->H[0], Hy = K->H[1], Hz = K->H[2];
  // rank-local apply buffers (unsharded: nz = Nz, nx = Px and X aliases A); the full octant
  // is built on every rank (it depends only on the grid and k)
  const size_t nA = size_t(Px) * Ny * K->nz, nB = size_t(K->nx) * Py * K->bz;
  // folded kx rows this kernel's kx columns [x0, x0 + nx) need (all Hx when unsharded)
  {
    int lo = Hx, hi = -1;
    for (int kx = K->x0; kx < K->x0 + K->nx; ++kx) {
      const int f = fusg::fold_index(kx, Px);
      lo = std::min(lo, f);
      hi = std::max(hi, f);
    }
    K->kf0 = hi < lo ? 0 : lo;
    K->knf = hi < lo ? 0 : hi - lo + 1;
  }
  const int kf0 = K->kf0, knf = K->knf;
  const size_t nK = size_t(std::max(knf, 1)) * Hy * Hz;
  const size_t nX = (K->G > 1 || K->slab) ? size_t(K->nx) * Nz * Ny : 0;
  // stream-ordered allocations: the context's pool keeps freed workspaces for the next kernel
  // (a cascade builds one GreenKernel per harmonic)
  cudaStream_t as = K->ctx->stream;
  double2 *g1 = nullptr, *g2 = nullptr;  // build scratch: [oz][oy][kx] and [oz][ky][kx] half-ranges
  // slab kernels: the A and x-slab buffers are peer-store targets, exported with CUDA IPC,
  // which needs cudaMalloc (not the stream-ordered pool)
  K->ipc_bufs = K->slab;
  auto alloc_ipc = [&](double2** p, size_t n) {
    return K->ipc_bufs ? cudaMalloc(p, n * sizeof(double2)) : cudaMallocAsync(p, n * sizeof(double2), as);
  };
  if (alloc_ipc(&K->bufA, nA) != cudaSuccess ||
      cudaMallocAsync(&K->bufB, nB * sizeof(double2), as) != cudaSuccess ||
      cudaMallocAsync(&K->koct, nK * sizeof(double2), as) != cudaSuccess ||
      (nX && alloc_ipc(&K->xbuf, nX) != cudaSuccess)) {
    cudaGetLastError();
    return set_error(FUSG_OOM, "GreenKernel: device allocation failed");
  }
  // build scratch: the apply workspaces are idle during the build, so G1/G2 live in bufA/bufB
  // whenever they fit (always unsharded) -- the peak stays at the apply's own footprint, which
  // is what lets a 1024^3 grid (2048^3 embedding) fit in one B200
  // G1 and G2 hold only the kx window [kf0, kf0 + knf) (compact, row stride knf; all Hx rows
  // unsharded): the x pass still transforms every (oy, oz) line but stores the window
  const size_t n1 = size_t(std::max(knf, 1)) * Ny * Nz, n2 = size_t(std::max(knf, 1)) * Hy * Nz;
  const bool g1_in_A = n1 <= nA, g2_in_B = n2 <= nB;
  g1 = g1_in_A ? K->bufA : nullptr;
  g2 = g2_in_B ? K->bufB : nullptr;
  if ((!g1_in_A && cudaMallocAsync(&g1, n1 * sizeof(double2), as) != cudaSuccess) ||
      (!g2_in_B && cudaMallocAsync(&g2, n2 * sizeof(double2), as) != cudaSuccess)) {
    cudaGetLastError();
    if (g1 && !g1_in_A) cudaFreeAsync(g1, as);
    return set_error(FUSG_OOM, "GreenKernel: build scratch allocation failed");
  }
  // (the all-to-all staging buffer rbuf, nX elements, is allocated by the first NCCL-transport
  // apply: the fused peer-store transport never needs it)
  K->bytes = (nA + nB + nK + nX) * sizeof(double2);

  fusg_ctx* ctx = K->ctx;
  cudaStream_t s = ctx->stream;
  const double dx = K->grid.dx;
  // G1: generate K along x for offsets (oy, oz) >= 0, forward x, keep kx <= Px/2
  KGenF gen{Nx, Ny, Px, dx, dx * dx * dx, K->k.k_re, K->k.k_im, self};
  GStoreF s1{GStore{g1, std::max(knf, 1), 0, 1, kf0 + knf, 1.0, kf0}};
  FUSG_TRY(launch_axis<false>(ctx, K->plan[0], Ny * Nz, 1, gen, s1, s));
  // G2: even extension along y, forward y, keep ky <= Py/2 (kx rows [kf0, kf0 + knf) only:
  // the y and z transforms are independent per kx, so an x-slab kernel builds just its window;
  // the x pass above is the replicated part of a sharded build, and no collective is needed)
  if (knf > 0) {
    FoldF l2{g1, 1, int64_t(Ny) * knf, knf, Ny, Py};
    GStoreF s2{GStore{g2, 1, int64_t(Hy) * knf, knf, Hy, 1.0}};
    FUSG_TRY(launch_axis<false>(ctx, K->plan[1], knf, Nz, l2, s2, s));
    // G3: even extension along z, forward z, keep kz <= Pz/2 -> octant rows [kf0, kf0 + knf)
    FoldF l3{g2, 1, knf, int64_t(Hy) * knf, Nz, Pz};
    GStoreF s3{GStore{K->koct, int64_t(Hy) * Hz, Hz, 1, Hz, 1.0}};  // octant [kx - kf0][ky][kz]
    FUSG_TRY(launch_axis<false>(ctx, K->plan[2], knf, Hy, l3, s3, s));
  }
  if (!g1_in_A) cudaFreeAsync(g1, s);
  if (!g2_in_B) cudaFreeAsync(g2, s);
  FUSG_CUDA_TRY(cudaStreamSynchronize(s));
  return FUSG_OK;
}

// ---------------------------------------------------------------------------- apply
// ---------------------------------------------------------------------------- apply phases
// Rank r of G owns z-planes [z0, z0 + nz) of f/u and, in spectral space, columns
// [x0, x0 + nx) of kx (unsharded: G = 1, nz = Nz, nx = Px, X == A).
//   phase A : f_r [nz][Ny][Nx] -> A_r [Px][nz][Ny]            (pass A; slices of A_r by kx
//             range are the all-to-all send blocks, contiguous)
//   exchange: A_r -> X_r [nx][Nz][Ny]                          (transpose z-slab -> x-slab)
//   phase BCD: X_r -> B_r [nx][Py][Nz] -> C in place -> X_r     (passes B, C, D)
//   exchange: X_r -> A_r                                       (transpose back)
//   phase E : A_r -> u_r                                       (pass E, scale/|P|, crop)
fusg_status apply_phase_A(fusg_kernel* K, const double2* f, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1];
  const int Px = K->P[0], nz = K->nz;
  return launch_axis<false>(K->ctx, K->plan[0], Ny, nz,
                            GLoadF{GLoad{f, Nx, int64_t(Ny) * Nx, 1, Nx}},
                            GStoreF{GStore{K->bufA, 1, K->az, K->akx, Px, 1.0}}, s, kKindRow);
}

// FUSG_CONV_QUAD=1: pass-C lines in quad order (kx mirror pairs interleaved at the finest
// level, conv_line_coords in warp_args.cuh) instead of kx-slow order.  Measured neutral to
// slightly slower (512: 0.703 -> 0.711 ms, 768: 2.88 -> 2.90, 1536: 34.0 -> 34.0), so off.
static int conv_quad() {
  static const int q = [] {
    const char* e = getenv("FUSG_CONV_QUAD");
    return (e && atoi(e) != 0) ? 1 : 0;
  }();
  return q;
}

// passes B, C on the x-slab X [nx][Nz][Ny] into B (ev, optional: marks after B and after C)
static fusg_status phase_BC(fusg_kernel* K, double2* X, cudaStream_t s, cudaEvent_t* ev) {
  const int Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1], Pz = K->P[2];
  const int Hy = K->H[1], Hz = K->H[2];
  const int nx = K->nx;
  const int64_t bz = K->bz, PyBz = int64_t(Py) * bz;
  // X: [kx][z][y] (x-slab) or A in the kernel's layout (unsharded)
  const int64_t xz = X == K->bufA ? K->az : Ny, xkx = X == K->bufA ? K->akx : int64_t(Nz) * Ny;
  FUSG_TRY(launch_axis<false>(K->ctx, K->plan[1], Nz, nx, GLoadF{GLoad{X, xz, xkx, 1, Ny}},
                              GStoreF{GStore{K->bufB, 1, PyBz, bz, Py, 1.0}}, s, kKindRow));
  if (ev) cudaEventRecord(ev[0], s);
  FUSG_TRY(launch_conv(K->ctx, K->plan[2], Py, nx, GLoadF{GLoad{K->bufB, bz, PyBz, 1, Nz}},
                       GStoreF{GStore{K->bufB, bz, PyBz, 1, Nz, 1.0}},
                       KOct{K->koct, Px, Py, Pz, int64_t(Hy) * Hz, Hz, 1, K->x0, conv_quad(), K->kf0}, s));
  if (ev) cudaEventRecord(ev[1], s);
  return FUSG_OK;
}

fusg_status apply_phase_BC(fusg_kernel* K, double2* X, cudaStream_t s) { return phase_BC(K, X, s, nullptr); }

// Fused transposes of the sharded apply: pass A stores each kx segment into the x-slab of the
// rank owning kx, pass D each z-row into the A slab of the rank owning z (PeerMap).  Both need
// the transposing warp kernels (padded x / y lengths with a warp-engine entry).
fusg_status apply_phase_A_peers(fusg_kernel* K, const double2* f, const PeerMap& pm, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  WArgs a{f, Nx, int64_t(Ny) * Nx, 1, Nx, nullptr, 1, Ny, int64_t(Nz) * Ny, K->P[0], 1.0,
          Ny, K->nz, K->plan[0].tw, KOct{}, pm};
  int r = K->P[0] == 512 ? launch_transpose_r16(K->ctx, true, a, s)
          : K->P[0] == 1536 ? launch_transpose_r16x3(K->ctx, true, a, s)
          : K->P[0] == 1024 ? launch_transpose_r16x2(K->ctx, true, a, s) : 0;
  if (r == 0) r = launch_mw(K->ctx, K->P[0], true, a, s);
  if (r == 0) r = launch_warp(K->ctx, K->P[0], kWRowToCol, false, a, s);
  if (r < 0) return FUSG_CUDA;
  if (r == 0) return set_error(FUSG_INVALID_ARGUMENT, "fused transposes need a padded x length of 256, 512, 768, 1024 or 1536");
  return FUSG_OK;
}

fusg_status apply_phase_D_peers(fusg_kernel* K, const PeerMap& pm, cudaStream_t s) {
  const int Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Py = K->P[1];
  const int64_t PyBz = int64_t(Py) * K->bz;
  WArgs a{K->bufB, 1, PyBz, K->bz, Py, nullptr, Ny, 0, 1, Ny, 1.0, Nz, K->nx, K->plan[1].tw, KOct{}, pm};
  int r = Py == 512 ? launch_transpose_r16(K->ctx, false, a, s)
          : Py == 1536 ? launch_transpose_r16x3(K->ctx, false, a, s)
          : Py == 1024 ? launch_transpose_r16x2(K->ctx, false, a, s) : 0;
  if (r == 0) r = launch_mw(K->ctx, Py, false, a, s);
  if (r == 0) r = launch_warp(K->ctx, Py, kWColToRow, true, a, s);
  if (r < 0) return FUSG_CUDA;
  if (r == 0) return set_error(FUSG_INVALID_ARGUMENT, "fused transposes need a padded y length of 256, 512, 768, 1024 or 1536");
  return FUSG_OK;
}

// passes B, C, D on the x-slab X [nx][Nz][Ny]; ev (optional) marks after B and after C
fusg_status apply_phase_BCD(fusg_kernel* K, double2* X, cudaStream_t s, cudaEvent_t* ev) {
  const int Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Py = K->P[1];
  const int nx = K->nx;
  const int64_t PyBz = int64_t(Py) * K->bz;
  const int64_t xz = X == K->bufA ? K->az : Ny, xkx = X == K->bufA ? K->akx : int64_t(Nz) * Ny;
  FUSG_TRY(phase_BC(K, X, s, ev));
  // D: ky columns of B (lines z, tiled, contiguous; outer kx) -> y rows of X, keep Ny
  return launch_axis<true>(K->ctx, K->plan[1], Nz, nx, GLoadF{GLoad{K->bufB, 1, PyBz, K->bz, Py}},
                           GStoreF{GStore{X, xz, xkx, 1, Ny, 1.0}}, s, kKindCol);
}

fusg_status apply_phase_E(fusg_kernel* K, double2* u, double scale, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1];
  const int Px = K->P[0], nz = K->nz;
  const double total = double(K->P[0]) * double(K->P[1]) * double(K->P[2]);
  (void)nz;
  return launch_axis<true>(K->ctx, K->plan[0], Ny, nz,
                           GLoadF{GLoad{K->bufA, 1, K->az, K->akx, Px}},
                           GStoreF{GStore{u, Nx, int64_t(Ny) * Nx, 1, Nx, scale / total}}, s, kKindCol);
}

// z-chunks of the unsharded apply.  Pass A and B lines never mix z-planes and neither do
// passes D and E, so a chunk of planes runs through A+B as soon as its input has arrived and
// through D+E as soon as pass C is done, while other chunks are still being copied.
fusg_status apply_chunk_AB(fusg_kernel* K, const double2* f_z0, int z0, int nzc, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1];
  const int64_t PyBz = int64_t(Py) * K->bz;
  (void)Nz;
  double2* A = K->bufA + int64_t(z0) * K->az;
  FUSG_TRY(launch_axis<false>(K->ctx, K->plan[0], Ny, nzc, GLoadF{GLoad{f_z0, Nx, int64_t(Ny) * Nx, 1, Nx}},
                              GStoreF{GStore{A, 1, K->az, K->akx, Px, 1.0}}, s, kKindRow));
  return launch_axis<false>(K->ctx, K->plan[1], nzc, Px, GLoadF{GLoad{A, K->az, K->akx, 1, Ny}},
                            GStoreF{GStore{K->bufB + z0, 1, PyBz, K->bz, Py, 1.0}}, s, kKindRow);
}

fusg_status apply_phase_C(fusg_kernel* K, cudaStream_t s) {
  const int Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1], Pz = K->P[2];
  const int64_t bz = K->bz, PyBz = int64_t(Py) * bz;
  return launch_conv(K->ctx, K->plan[2], Py, Px, GLoadF{GLoad{K->bufB, bz, PyBz, 1, Nz}},
                     GStoreF{GStore{K->bufB, bz, PyBz, 1, Nz, 1.0}},
                     KOct{K->koct, Px, Py, Pz, int64_t(K->H[1]) * K->H[2], K->H[2], 1, 0, conv_quad(), K->kf0}, s);
}

fusg_status apply_chunk_DE(fusg_kernel* K, double2* u_z0, int z0, int nzc, double scale, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1];
  const int64_t PyBz = int64_t(Py) * K->bz;
  const double total = double(K->P[0]) * double(K->P[1]) * double(K->P[2]);
  (void)Nz;
  double2* A = K->bufA + int64_t(z0) * K->az;
  FUSG_TRY(launch_axis<true>(K->ctx, K->plan[1], nzc, Px, GLoadF{GLoad{K->bufB + z0, 1, PyBz, K->bz, Py}},
                             GStoreF{GStore{A, K->az, K->akx, 1, Ny, 1.0}}, s, kKindCol));
  return launch_axis<true>(K->ctx, K->plan[0], Ny, nzc, GLoadF{GLoad{A, 1, K->az, K->akx, Px}},
                           GStoreF{GStore{u_z0, Nx, int64_t(Ny) * Nx, 1, Nx, scale / total}}, s, kKindCol);
}

// Passes A and B as one launch through an L2-resident ring (conv_r16.cu): unsharded applies
// with Px = Py = 512 and pruned x / y halves (the 16 x 16 x 2 kernels), ring slot <= 24 MB.
// The ring lives in the head of bufA, which pass D overwrites afterwards.  1 done, 0 n/a.
static int try_ab_fused(fusg_kernel* K, const double2* f, cudaStream_t s) {
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1];
  if (K->G != 1 || K->slab || Px != 512 || Py != 512 || 2 * Nx > Px || 2 * Ny > Py) return 0;
  if (K->az != Ny) return 0;  // the ring assumes A as [kx][z][y]
  constexpr int kRing = 3;
  const int64_t slot = int64_t(Px) * 8 * Ny;
  if (slot * int64_t(sizeof(double2)) > (int64_t(24) << 20) || kRing * slot > int64_t(Px) * Nz * Ny) return 0;
  const int slabs = (Nz + 7) / 8;
  if (!K->absync && cudaMalloc(&K->absync, sizeof(int) * (1 + 2 * 4096)) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (slabs > 4096) return 0;
  const int64_t PyBz = int64_t(Py) * K->bz;
  ABFused fa;
  fa.a = WArgs{f, Nx, int64_t(Ny) * Nx, 1, Nx, K->bufA, 1, Ny, 8 * int64_t(Ny), Px, 1.0, Ny, Nz, K->plan[0].tw, KOct{}};
  fa.b = WArgs{K->bufA, Ny, 8 * int64_t(Ny), 1, Ny, K->bufB, 1, PyBz, K->bz, Py, 1.0, 8, Px, K->plan[1].tw, KOct{}};
  fa.nz = Nz;
  fa.slabs = slabs;
  fa.ring = kRing;
  fa.slot = slot;
  fa.sync = K->absync;
  return launch_ab_fused_r16(K->ctx, fa, s);
}

// Passes A and B z-chunk by z-chunk on two streams (FUSG_AB_CHUNKS=1): pass A of chunk c
// (8 planes) writes ring slot c % R (R = 3, 16 MB each at cfg2, the head of bufA), pass B of
// chunk c reads it on a second stream while pass A of chunk c + 1 runs, and drops the slot's L2
// lines after reading them.  Regular (non-persistent) launches; events order the ring reuse.
// 1 done, 0 not applicable, -1 error.
static int try_ab_chunks(fusg_kernel* K, const double2* f, cudaStream_t s) {
  static const bool on = [] {
    const char* e = getenv("FUSG_AB_CHUNKS");
    return e && atoi(e) != 0;
  }();
  const int Nx = K->grid.dims[0], Ny = K->grid.dims[1], Nz = K->grid.dims[2];
  const int Px = K->P[0], Py = K->P[1];
  if (!on || K->G != 1 || K->slab || Px != 512 || Py != 512 || 2 * Nx > Px || 2 * Ny > Py) return 0;
  if (K->az != Ny) return 0;  // the ring assumes A as [kx][z][y]
  constexpr int kRing = 3;
  const int64_t slot = int64_t(Px) * 8 * Ny;
  if (kRing * slot > int64_t(Px) * Nz * Ny) return 0;
  const int C = (Nz + 7) / 8;
  if (!K->ab_stream && cudaStreamCreateWithFlags(&K->ab_stream, cudaStreamNonBlocking) != cudaSuccess)
    return -1;
  while (int(K->ab_ev.size()) < 2 * C + 1) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return -1;
    K->ab_ev.push_back(e);
  }
  cudaEvent_t* evA = K->ab_ev.data();  // evA[2c], evB[2c + 1], start = [2C]
  // the B stream starts after everything already queued on s (e.g. the previous apply)
  if (cudaEventRecord(K->ab_ev[2 * C], s) != cudaSuccess || cudaStreamWaitEvent(K->ab_stream, K->ab_ev[2 * C], 0))
    return -1;
  const int64_t PyBz = int64_t(Py) * K->bz;
  for (int c = 0; c < C; ++c) {
    const int z0 = 8 * c, nzc = std::min(8, Nz - z0);
    double2* const sl = K->bufA + int64_t(c % kRing) * slot;
    if (c >= kRing && cudaStreamWaitEvent(s, evA[2 * (c - kRing) + 1], 0) != cudaSuccess) return -1;
    const WArgs wa{f + int64_t(z0) * Nx * Ny, Nx, int64_t(Nx) * Ny, 1, Nx, sl, 1, Ny, 8 * int64_t(Ny), Px, 1.0,
                   Ny, nzc, K->plan[0].tw, KOct{}};
    if (launch_r16_chunk(K->ctx, false, wa, s) < 0) return -1;
    if (cudaEventRecord(evA[2 * c], s) != cudaSuccess || cudaStreamWaitEvent(K->ab_stream, evA[2 * c], 0))
      return -1;
    const WArgs wb{sl, Ny, 8 * int64_t(Ny), 1, Ny, K->bufB + z0, 1, PyBz, K->bz, Py, 1.0, nzc, Px, K->plan[1].tw,
                   KOct{}};
    if (launch_r16_chunk(K->ctx, true, wb, K->ab_stream) < 0) return -1;
    if (cudaEventRecord(evA[2 * c + 1], K->ab_stream) != cudaSuccess) return -1;
  }
  if (cudaStreamWaitEvent(s, evA[2 * (C - 1) + 1], 0) != cudaSuccess) return -1;
  return 1;
}

fusg_status volume_potential_apply(fusg_kernel* K, const double2* f, double2* u, double scale,
                                   cudaStream_t s, cudaEvent_t* ev) {
  if (K->G != 1) return set_error(FUSG_INVALID_ARGUMENT, "kernel_apply: sharded kernel needs a slab apply");
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
  };
  mark(0);
  int fused = try_ab_chunks(K, f, s);
  if (fused == 0) fused = try_ab_fused(K, f, s);
  if (fused < 0) return FUSG_CUDA;
  if (fused) {  // A+B in one launch (both marks after it), then C, D, E
    const int Ny = K->grid.dims[1], Nz = K->grid.dims[2];
    const int64_t PyBz = int64_t(K->P[1]) * K->bz;
    mark(1);
    mark(2);
    FUSG_TRY(apply_phase_C(K, s));
    mark(3);
    FUSG_TRY(launch_axis<true>(K->ctx, K->plan[1], Nz, K->P[0], GLoadF{GLoad{K->bufB, 1, PyBz, K->bz, K->P[1]}},
                               GStoreF{GStore{K->bufA, K->az, K->akx, 1, Ny, 1.0}}, s, kKindCol));
    mark(4);
    FUSG_TRY(apply_phase_E(K, u, scale, s));
    mark(5);
    return FUSG_OK;
  }
  FUSG_TRY(apply_phase_A(K, f, s));
  mark(1);
  FUSG_TRY(apply_phase_BCD(K, K->bufA, s, ev ? ev + 2 : nullptr));
  mark(4);
  FUSG_TRY(apply_phase_E(K, u, scale, s));
  mark(5);
  return FUSG_OK;
}

}  // namespace fusg
