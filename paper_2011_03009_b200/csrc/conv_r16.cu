// Pass C of the apply at padded z length 512 as a 16 x 16 x 2 transform per warp (see below).
#include <utility>
#include <cstdlib>
#include <algorithm>

#include "warp_args.cuh"
// the tan-form radix 2 inside the fused K^ multiply is a gain at 1536 only: here 0.705 vs 0.708 ms at cfg2
#ifndef FUSG_R2_TAN_MULK
#define FUSG_R2_TAN_MULK 0
#endif
#include "r16.cuh"

namespace fusg {

// Pass C at L = 512, pruned (Nz <= 256 in and out), as 512 = 16 x 16 x 2 on one warp:
//   stage A  radix 16 in registers over n1 (n = 32 n1 + n2, lane = n2), twiddle W512^(n2 k1);
//   exchange through shared memory (registers k1 -> registers n2hi, n2 = 2 n2hi + n2lo);
//   stage B  radix 16 in registers over n2hi, then the last radix 2 over n2lo ACROSS the lane
//            pair (lane, lane ^ 16) with one half-exchange of 8 values by warp shuffle.
// Against the radix-8 Stockham kernel (two shared exchanges per transform) this moves half the
// bytes through the L1/shared data pipe per line (one shared exchange + half a shuffle
// exchange), the unit that kernel saturates.  The inverse transform is the adjoint, so the
// spectrum stays in the half-exchanged layout for the K^ multiply and the inverse radix 2
// starts in-lane.  Layout after the forward transform: lane = 16 b + k1 holds, in slot i,
// X[k1 + 16 (i + 8 b)] and, in slot i + 8, X[k1 + 16 (i + 8 b) + 256].
// Exchange buffer: row k1 (32 entries), column n2 ^ (k1 & 7): both access patterns are
// bank-conflict-free (8 lanes of each 128-byte phase hit 8 distinct 16-byte bank groups).
// Pass C (FUSG_R16_PAD, default on): the exchange buffer as 16 rows of 33 entries instead, also
// conflict-free for both patterns and affine in the lane, so every offset folds into the
// instruction's immediate (the XOR costs a LOP3 per access).
#ifndef FUSG_R16_PAD
#define FUSG_R16_PAD 1
#endif
constexpr int kR16XL = FUSG_R16_PAD ? 16 * 33 : 512;  // exchange buffer entries per warp (pass C)
__device__ __forceinline__ int r16_exc(int row, int col) { return FUSG_R16_PAD ? row * 33 + col : r16_ex(row, col); }
// per-warp buffers of the radix-8 kernel + the CTA's twiddle bases
template <bool TAB>
constexpr size_t r16_smem_bytes(int nw, bool kl2 = false) {
  return size_t(nw) * (kR16XL - 512 + (kl2 ? 512 + PPConvSmem<512, true>::STAGE : PPConvSmem<512, true>::PER_WARP)) * sizeof(double2) +
         nw * 2 * sizeof(uint64_t) + (TAB ? 16 : 4) * 32 * sizeof(double2);
}

// KL2: the K^ row is not staged in shared memory; it is prefetched into L2 one line ahead
// (cp.async.bulk.prefetch) and read at the multiply with read-only loads.  12 KB per warp
// instead of 16 lets 16 warps share an SM (MINB 4, 128 registers).
// FULL: every row holds 256 valid inputs and outputs (cfg2): no predicates or zero fills
template <int NW, int MINB, bool TAB, bool KL2 = false, bool FULL = false>
__global__ void __launch_bounds__(NW * 32, MINB) warp_row_conv_r16(WArgs a) {
  constexpr int L = 512;
  constexpr int HZ = L / 2 + 1;
  using SM = PPConvSmem<L, true>;
  constexpr int PW = kR16XL - L + (KL2 ? L + SM::STAGE : SM::PER_WARP);  // double2 per warp
  extern __shared__ double2 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const xb = sm + size_t(w) * PW;
  double2* const sb = xb + kR16XL;
  double2* const kb = sb + SM::STAGE;  // (unused when KL2)
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + size_t(NW) * PW) + 2 * w;
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init_fence();
  }
  __syncwarp();
  unsigned ph_in = 0, ph_k = 0;
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t stride = int64_t(gridDim.x) * NW;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) {  // line < 2^31 (host-checked)
    conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx);
  };
  // (ky, kx) of a line costs ~45 instructions (divisions); each line's pair is computed once, one
  // line ahead, and serves both refills and the output row
  auto prefetch_in = [&](bool ok, int ky, int kx) {
    if (ok && lane == 0)
      bulk_stage(sb, a.in + ky * a.in_si + int64_t(kx) * a.in_sk, unsigned(a.in_nvalid) * sizeof(double2), bars);
  };
  auto prefetch_k = [&](bool ok, int ky, int kx) {
    if (ok && lane == 0) {
      if constexpr (KL2) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.ko.line(ky, kx)), "r"(unsigned(HZ * sizeof(double2)))
                     : "memory");
      } else {
        bulk_stage(kb, a.ko.line(ky, kx), HZ * sizeof(double2), bars + 1);
      }
    }
  };
  double2* const tws = sm + size_t(NW) * PW + NW;  // after the 2 NW mbarriers
  if (w == 0) {
    if constexpr (TAB) {
      for (int j = 0; j < 16; ++j) tws[32 * j + lane] = __ldg(a.tw + ((lane * j) & (L - 1)));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) tws[32 * j + lane] = __ldg(a.tw + ((lane << j) & (L - 1)));
    }
  }
  __syncthreads();
  const R16Tw<TAB> tw{tws, lane};
  const bool b = lane >= 16;
  const int k1 = lane & 15;
  const auto I8 = std::make_integer_sequence<int, 8>{};
  int64_t line = int64_t(blockIdx.x) * NW + w;
  int ky = 0, kx = 0;
  if (line < nlines) coords(line, ky, kx);
  prefetch_in(line < nlines, ky, kx);
  prefetch_k(line < nlines, ky, kx);
  for (; line < nlines; line += stride) {
    const bool more = line + stride < nlines;
    int kyn = 0, kxn = 0;
    if (more) coords(line + stride, kyn, kxn);
    mbar_wait(bars, ph_in);
    ph_in ^= 1;
    double2 v[16];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int pos = lane + 32 * e;
      v[e] = (FULL || pos < a.in_nvalid) ? sb[pos] : make_double2(0.0, 0.0);
    }
    __syncwarp();  // S consumed: refill it with the next line while this one is transformed
    prefetch_in(more, kyn, kxn);
    // forward stage A (upper half zero) and its twiddle
    dft16_half_in<false>(v);
    tw.apply<false>(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) xb[r16_exc(k, lane)] = v[k];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = xb[r16_exc(k1, 2 * h + int(b))];
    // forward stage B and the cross-lane radix 2
    dft16<false>(v);
    if constexpr (!KL2) {
      // the cross-lane radix 2 fused with the folded-K^ multiply (p < 256, mirror 256 - p)
      mbar_wait(bars + 1, ph_k);
      ph_k ^= 1;
      r16_fwd_r2_mulk_all<16, 256>(v, b, kb, k1 + 128 * int(b), I8);
      __syncwarp();  // K^ row consumed
      prefetch_k(more, kyn, kxn);
    } else {
      r16_r2_all<false>(v, b, I8);
    }
    if constexpr (KL2) {
      const double2* kl = a.ko.line(ky, kx);
      prefetch_k(more, kyn, kxn);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int p = k1 + 16 * (i + 8 * int(b));  // < 256; its mirror p + 256 folds to 256 - p
        v[i] = cmul(v[i], __ldg(kl + p));
        v[i + 8] = cmul(v[i + 8], __ldg(kl + 256 - p));
      }
    }
    // inverse: radix 2 (in-lane) + half-exchange back, stage B, exchange, twiddle, stage A
    r16_r2_all<true>(v, b, I8);
    dft16<true>(v);
#pragma unroll
    for (int h = 0; h < 16; ++h) xb[r16_exc(k1, 2 * h + int(b))] = v[h];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xb[r16_exc(k, lane)];
    tw.apply<true>(v);
    dft16_half_out<true>(v);
    double2* out = a.out + ky * a.out_si + int64_t(kx) * a.out_sk;
    ky = kyn;
    kx = kxn;
    if (a.scale == 1.0) {  // (always, inside the apply: the scale rides on pass E)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int pos = lane + 32 * e;
        if (FULL || pos < a.out_nvalid) out[pos] = v[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int pos = lane + 32 * e;
        if (FULL || pos < a.out_nvalid) out[pos] = cscale(v[e], a.scale);
      }
    }
    __syncwarp();  // every lane has read the exchange buffer before the next line writes it
  }
}


int launch_conv_r16(fusg_ctx* ctx, const WArgs& a, cudaStream_t s) {
  static const bool on = [] {  // FUSG_CONV_R16=0 selects the radix-8 Stockham pass C at 512
    const char* e = getenv("FUSG_CONV_R16");
    return !(e && atoi(e) == 0);
  }();
  if (!on || 2 * a.in_nvalid > 512 || 2 * a.out_nvalid > 512 || a.in_nvalid < 1) return 0;
  static const int tab = [] {  // FUSG_R16_TAB=1: all fifteen twiddles from the shared table
    const char* e = getenv("FUSG_R16_TAB");
    return e ? atoi(e) : 0;
  }();
  const int64_t nl = int64_t(a.n_inner) * a.n_outer;
  if (nl >= (int64_t(1) << 31)) return 0;
  static const int nw = [] {  // FUSG_R16_NW: warps per CTA (2, 3, 4, 6; 12 warps per SM)
    const char* e = getenv("FUSG_R16_NW");
    const int v = e ? atoi(e) : 4;
    return (v == 2 || v == 3 || v == 6) ? v : 4;
  }();
  static const int kl2 = [] {  // FUSG_R16_KL2=1: K^ rows through L2, 16 warps per SM
    const char* e = getenv("FUSG_R16_KL2");
    return e ? atoi(e) : 0;
  }();
  using Fn = void (*)(WArgs);
  const Fn fn = kl2 ? warp_row_conv_r16<4, 4, false, true>
                : nw == 2 ? (tab ? warp_row_conv_r16<2, 6, true> : warp_row_conv_r16<2, 6, false>)
                : nw == 3 ? (tab ? warp_row_conv_r16<3, 4, true> : warp_row_conv_r16<3, 4, false>)
                : nw == 6 ? (tab ? warp_row_conv_r16<6, 2, true> : warp_row_conv_r16<6, 2, false>)
                : (!tab && a.in_nvalid == 256 && a.out_nvalid == 256) ? warp_row_conv_r16<4, FUSG_PP_MINB, false, false, true>
                          : (tab ? warp_row_conv_r16<4, FUSG_PP_MINB, true> : warp_row_conv_r16<4, FUSG_PP_MINB, false>);
  const size_t smem = kl2 ? r16_smem_bytes<false>(4, true) : tab ? r16_smem_bytes<true>(nw) : r16_smem_bytes<false>(nw);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
    set_error(FUSG_CUDA, "pass C (16x16x2): cannot configure shared memory");
    return -1;
  }
  int per_sm = 0;
  const int nwl = kl2 ? 4 : nw;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nwl * 32, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  const int64_t lines = int64_t(a.n_inner) * a.n_outer;
  // FUSG_R16_WAVES: CTAs per resident slot (1 = fully persistent).  8 measured best on cfg2
  // (0.730 -> 0.687 ms): CTAs retiring and relaunching through the block scheduler keep the
  // SMs' warps out of phase better than one long-lived CTA per slot.
  static const int waves = [] {
    const char* e = getenv("FUSG_R16_WAVES");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const int64_t grid = std::min<int64_t>((lines + nwl - 1) / nwl, int64_t(per_sm) * ctx->num_sms * waves);
  fn<<<unsigned(grid), nwl * 32, smem, s>>>(a);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "pass C (16x16x2)");
    return -1;
  }
  return 1;
}

// ---------------------------------------------------------------------------- transposing passes
// Passes A/B (forward, zero-padded upper input half) and D/E (inverse, cropped upper output
// half) at L = 512 on the same 16 x 16 x 2 warp transform.

// A/B: a CTA owns 8 adjacent rows (i0..i0+7 at outer k), warp w transforms row w read straight
// from global memory (512 B per warp instruction), exchanges in place in column w of the
// swizzled [pos][8] tile, leaves its spectrum there, and after one CTA barrier the CTA stores
// positions as 8 adjacent lines (128 contiguous bytes).
constexpr size_t kR16TileBytes = size_t(512) * 8 * sizeof(double2);

// L2 eviction-priority hints for the fused A+B pass: the streamed input f and output B are
// evict-first so they do not push the ring out of L2; ring stores are evict-last.
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_nc_hint(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void l2_discard(const void* p) {  // drop a dead 128-byte line, no write-back
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// Input / output access modes of r2c_tile: plain (__ldg, st), fused-pass reads of f (evict-first)
// and of the ring (ld.global.cg: written by other CTAs of the launch), stores to the ring
// (evict-last) and to B (evict-first).
enum R2CMode { kR2CPlain = 0, kR2CFusedA = 1, kR2CFusedB = 2 };

// One 8-row tile (rows i0..i0+7 at outer k) of a row -> column pass; CG: read the input rows
// through L2 only (ld.global.cg: rows another CTA of the same launch wrote).
// (in_base, out_base, n_inner override a's for the fused A+B kernel.)
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// stage (optional): the tile's input rows already staged in shared memory, row w at
// stage + w * a.in_si; after_load() runs once every warp has its row in registers (after a CTA
// barrier), so the caller may refill the stage while the tile is transformed.
template <int MODE, class Hook = NoHook>
__device__ __forceinline__ void r2c_tile(const WArgs& a, const double2* in_base, double2* out_base, int n_inner,
                                         int i0, int k, double2* tile, bool hints = true,
                                         const double2* stage = nullptr, Hook after_load = Hook{}) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lines_ok = min(8, n_inner - i0);
  const bool ok = w < lines_ok;
  const double2* in = in_base + int64_t(i0 + (ok ? w : 0)) * a.in_si + int64_t(k) * a.in_sk;
  double2 v[16];
  const uint64_t pol_first = MODE != kR2CPlain ? l2_policy_first() : 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int pos = lane + 32 * e;
    v[e] = make_double2(0.0, 0.0);
    if (ok && pos < a.in_nvalid) {
      if (stage) v[e] = stage[w * a.in_si + pos];
      else
        v[e] = MODE == kR2CFusedB ? __ldcg(in + pos)
               : (MODE == kR2CFusedA && hints) ? ld_nc_hint(in + pos, pol_first) : __ldg(in + pos);
    }
  }
  if (stage) {
    __syncthreads();  // every warp has its row: the stage may be refilled
    after_load();
  }
  dft16_half_in<false>(v);
  {  // one exact table power per lane, the others by squaring (one FFT per warp)
    const double2 w1 = __ldg(a.tw + lane), w2 = cmul(w1, w1), w4 = cmul(w2, w2);
    r16_twiddle<false>(v, w1, w2, w4, cmul(w4, w4));
  }
  const bool b = lane >= 16;
  const int k1 = lane & 15;
#pragma unroll
  for (int q = 0; q < 16; ++q) tile[tile_at(r16_ex(q, lane), w)] = v[q];
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 16; ++h) v[h] = tile[tile_at(r16_ex(k1, 2 * h + int(b)), w)];
  dft16<false>(v);
  r16_r2_all<false>(v, b, std::make_integer_sequence<int, 8>{});
  __syncwarp();  // every lane has read its exchange slots
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int p = k1 + 16 * (i + 8 * int(b));
    tile[tile_at(p, w)] = v[i];
    tile[tile_at(p + 256, w)] = v[i + 8];
  }
  __syncthreads();
  if (a.pm.n == 0) {
    double2* base = out_base + int64_t(i0) * a.out_si + int64_t(k) * a.out_sk;
    const uint64_t pol = MODE == kR2CFusedA ? l2_policy_last() : pol_first;
#pragma unroll 4
    for (int e = threadIdx.x; e < a.out_nvalid * 8; e += 256) {
      const int pos = e >> 3, t = e & 7;
      if (t < lines_ok) {
        const double2 x = tile[tile_at(pos, t)];
        const double2 y = (a.scale == 1.0) ? x : cscale(x, a.scale);
        if (MODE == kR2CPlain || !hints) base[t * a.out_si + pos * a.out_sp] = y;
        else st_hint(base + t * a.out_si + pos * a.out_sp, y, pol);
      }
    }
  } else {  // fused transpose: the segment of position pos (kx) goes straight to the rank owning it
    for (int e = threadIdx.x; e < a.out_nvalid * 8; e += 256) {
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

__global__ void __launch_bounds__(256, 2) warp_row_to_col_r16(WArgs a) {
  extern __shared__ double2 tile[];
  const unsigned ntiles = unsigned(a.n_inner + 7) / 8u;
  const unsigned kq = blockIdx.x / ntiles;
  r2c_tile<kR2CPlain>(a, a.in, a.out, a.n_inner, int(blockIdx.x - kq * ntiles) * 8, int(kq), tile);
}

// Pass B of one z-chunk read from an L2-resident ring slot [kx][zz][y] (CTA = one kx, all zz):
// after the tile is stored, its input block is dead and its L2 lines are dropped without
// write-back (the slot is rewritten by a later chunk's pass A).
__global__ void __launch_bounds__(256, 2) warp_row_to_col_r16_ring(WArgs a) {
  extern __shared__ double2 tile[];
  const int k = blockIdx.x;  // n_inner <= 8: one tile per kx
  r2c_tile<kR2CPlain>(a, a.in, a.out, a.n_inner, 0, k, tile);
  const char* blk = reinterpret_cast<const char*>(a.in + int64_t(k) * a.in_sk);
  const int lines = int((int64_t(a.n_inner) * a.in_si * int64_t(sizeof(double2)) + 127) / 128);
  for (int l = threadIdx.x; l < lines; l += 256) l2_discard(blk + 128 * l);
}

// Passes A and B of a z-chunk on two streams through ring slot buffers (volume_potential.cu):
// pass A of the chunk (rows of f -> slot) or pass B (slot -> B).  1 launched, -1 error.
int launch_r16_chunk(fusg_ctx* ctx, bool pass_b, const WArgs& a, cudaStream_t s) {
  const auto fn = pass_b ? warp_row_to_col_r16_ring : warp_row_to_col_r16;
  static std::atomic<uint64_t> attr_mask{0};
  const bool attr = once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(warp_row_to_col_r16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(kR16TileBytes)) == cudaSuccess &&
           cudaFuncSetAttribute(warp_row_to_col_r16_ring, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(kR16TileBytes)) == cudaSuccess;
  });
  if (!attr) {
    set_error(FUSG_CUDA, "z-chunk A/B: cannot configure shared memory");
    return -1;
  }
  const unsigned blocks = pass_b ? unsigned(a.n_outer) : unsigned((a.n_inner + 7) / 8) * unsigned(a.n_outer);
  fn<<<blocks, 256, kR16TileBytes, s>>>(a);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "z-chunk A/B");
    return -1;
  }
  return 1;
}

// Passes A and B fused through an L2-resident ring of z-slabs (8 planes each).  Pass A of slab
// s writes its [kx][8][y] block into ring slot s % R; pass B of slab s reads it back (through
// L2) as soon as every pass-A tile of the slab is done.  The ring replaces the full [kx][z][y]
// intermediate, whose HBM write and read-back were a third of the A + B traffic.
// Persistent CTAs take work items from a global ticket in the order A(0), A(1), B(0), A(2),
// B(1), ..., B(S-1); B(s) waits for A(s) to finish and A(s) (s >= R) for B(s - R), both
// dispatched earlier, so the waits cannot deadlock.


__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Work item t of the fused A+B order A(0) | [A(p), B(p-1)], p = 1..S-1 | B(S-1): kind, slab s,
// index r within the slab's items, and the counter / count it waits for (none: dep = nullptr).
struct ABItem {
  bool isA;
  int s, r;
  const int* dep;
  int need;
};
__device__ __forceinline__ ABItem ab_item(const ABFused& f, int t) {
  const int nyt = (f.a.n_inner + 7) / 8, nkx = f.b.n_outer, S = f.slabs;
  const int last_nz = f.nz - 8 * (S - 1);
  const int na_full = nyt * 8, na_last = nyt * last_nz;
  ABItem it;
  if (f.mode & 16) {  // experiment: every A item, then every B item (ring = one slot per slab)
    const int na = nyt * f.nz;
    if (t < na) {
      it.isA = true, it.s = t / na_full, it.r = t - it.s * na_full, it.dep = nullptr, it.need = 0;
    } else {
      const int u = t - na;
      it.isA = false, it.s = u / nkx, it.r = u - it.s * nkx;
      it.dep = f.sync + 1 + it.s;
      it.need = it.s == S - 1 ? na_last : na_full;
    }
    return it;
  }
  const int a0 = S == 1 ? na_last : na_full;
  if (t < a0) {
    it.isA = true, it.s = 0, it.r = t;
  } else {
    const int rem = t - a0;
    const int full = na_full + nkx;  // groups p = 1..S-2: A(p) (full slab) then B(p-1)
    const int nfull = S >= 2 ? S - 2 : 0;
    if (rem < nfull * full) {
      const int p = 1 + rem / full, r = rem - (p - 1) * full;
      if (r < na_full) it.isA = true, it.s = p, it.r = r;
      else it.isA = false, it.s = p - 1, it.r = r - na_full;
    } else {
      int r = rem - nfull * full;
      if (S >= 2 && r < na_last) {  // A(S-1), the ragged last slab
        it.isA = true, it.s = S - 1, it.r = r;
      } else {
        if (S >= 2) r -= na_last;
        if (S >= 2 && r < nkx) it.isA = false, it.s = S - 2, it.r = r;
        else it.isA = false, it.s = S - 1, it.r = S >= 2 ? r - nkx : r;
      }
    }
  }
  if (it.isA) {  // the ring slot must have been read out by B(s - R)
    it.dep = it.s >= f.ring ? f.sync + 1 + S + (it.s - f.ring) : nullptr;
    it.need = nkx;
  } else {  // every pass-A tile of the slab must be in the ring
    it.dep = f.sync + 1 + it.s;
    it.need = it.s == S - 1 ? na_last : na_full;
  }
  return it;
}

// Persistent CTAs take items round-robin (CTA c: c, c + G, ...), all co-resident.  The
// smallest unfinished item's dependencies all have smaller indices, so some CTA can always
// progress.  Each item's input is one contiguous block (8 rows of f, or the ring block
// [kx][zz][y] of one kx), copied into a 32 KB shared stage by one 1-D bulk copy (TMA); the next
// item's copy is issued as soon as the current rows are in registers (if its dependency is
// already met, else at its start).  Completions are published by thread 0 after a CTA barrier
// (fence + add).
constexpr int kABStage = 8 * 256;  // staged input elements (8 rows of <= 256)
constexpr size_t kABFusedBytes = kR16TileBytes + kABStage * sizeof(double2) + 16;

__global__ void __launch_bounds__(256, 2) ab_fused_r16(ABFused f) {
  extern __shared__ double2 sm[];
  double2* const tile = sm;
  double2* const stage = sm + 512 * 8;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(stage + kABStage);
  const int nyt = (f.a.n_inner + 7) / 8;
  const int last_nz = f.nz - 8 * (f.slabs - 1);
  const int total = nyt * f.nz + f.b.n_outer * f.slabs;
  int* const doneA = f.sync + 1;
  int* const doneB = f.sync + 1 + f.slabs;
  auto slot_of = [&](int s) { return const_cast<double2*>(f.b.in) + int64_t(s % f.ring) * f.slot; };
  // thread 0: issue the bulk copy of item it's input block
  auto issue = [&](const ABItem& it) {
    const double2* src;
    unsigned bytes;
    if (it.isA) {
      const int zz = it.r / nyt, y0 = (it.r - zz * nyt) * 8;
      src = f.a.in + int64_t(y0) * f.a.in_si + int64_t(8 * it.s + zz) * f.a.in_sk;
      bytes = unsigned(min(8, f.a.n_inner - y0) * f.a.in_si * sizeof(double2));
    } else {
      const int nzs = it.s == f.slabs - 1 ? last_nz : 8;
      src = slot_of(it.s) + int64_t(it.r) * f.b.in_sk;
      bytes = unsigned(nzs * f.b.in_si * sizeof(double2));
      asm volatile("fence.proxy.async.global;" ::: "memory");  // ring rows written by generic stores
    }
    bulk_stage(stage, src, bytes, bar);
  };
  // thread 0: is item it's input dependency met (B: its slab's pass-A tiles all done)?
  auto input_ready = [&](const ABItem& it, bool wait) {
    if (it.isA) return true;
    if (wait) {
      while (ld_acquire(doneA + it.s) < it.need) __nanosleep(32);
      return true;
    }
    if (ld_relaxed(doneA + it.s) < it.need) return false;
    __threadfence();  // acquire side of the observation
    return true;
  };
  bool pre = false;     // thread 0: the current item's input copy is already in flight
  int* pub = nullptr;   // thread 0: counter of the finished item not yet published
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init_fence();
    if (int(blockIdx.x) < total) {
      const ABItem it = ab_item(f, blockIdx.x);
      pre = input_ready(it, false);
      if (pre) issue(it);
    }
  }
  __syncthreads();
  unsigned phase = 0;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const ABItem it = ab_item(f, t);
    if (threadIdx.x == 0) {
      if (pub && (!pre || (it.isA && it.dep))) {  // about to block: publish first (no self-wait)
        if (!(f.mode & 2)) __threadfence();
        atomicAdd(pub, 1);
        pub = nullptr;
      }
      if (!pre) {
        input_ready(it, true);
        issue(it);
      }
      if (it.isA && it.dep)  // the ring slot must have been read out by B(s - R)
        while (ld_acquire(it.dep) < it.need) __nanosleep(32);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    double2* const slot = slot_of(it.s);
    const int nzs = it.s == f.slabs - 1 ? last_nz : 8;
    auto refill = [&]() {  // after the CTA barrier in r2c_tile: the stage is free
      if (threadIdx.x == 0) {
        if (pub) {  // the previous item's stores were all issued before this barrier
          if (!(f.mode & 2)) __threadfence();
          atomicAdd(pub, 1);
          pub = nullptr;
        }
        pre = false;
        const int tn = t + int(gridDim.x);
        if (tn < total) {
          const ABItem nx = ab_item(f, tn);
          pre = input_ready(nx, false);
          if (pre) issue(nx);
        }
      }
      if (!it.isA && !(f.mode & 4)) {
        // the ring block [kx = r][zz < nzs][y] is dead (this item's rows are in registers): drop
        // its L2 lines without write-back
        const char* blk = reinterpret_cast<const char*>(slot + int64_t(it.r) * f.b.in_sk);
        const int lines = int((int64_t(nzs) * f.b.in_si * int64_t(sizeof(double2)) + 127) / 128);
        for (int l = threadIdx.x; l < lines; l += 256) l2_discard(blk + 128 * l);
      }
    };
    if (it.isA) {
      const int zz = it.r / nyt, yt = it.r - zz * nyt;
      // k = z indexes f; in the slot it is z - 8 s
      r2c_tile<kR2CFusedA>(f.a, f.a.in, slot - int64_t(8 * it.s) * f.a.out_sk, f.a.n_inner, yt * 8,
                           8 * it.s + zz, tile, !(f.mode & 8), stage, refill);
    } else {
      r2c_tile<kR2CFusedB>(f.b, slot, f.b.out + 8 * it.s, nzs, 0, it.r, tile, !(f.mode & 8), stage, refill);
    }
    // publication is deferred to the next item's refill barrier (or the end); the tile is
    // reused by the next item only after its own exchange barriers
    if (threadIdx.x == 0) pub = it.isA ? doneA + it.s : doneB + it.s;  // B: also its discards
    __syncthreads();  // the tile's cooperative reads are done before the next item writes it
  }
  if (threadIdx.x == 0 && pub) {
    if (!(f.mode & 2)) __threadfence();
    atomicAdd(pub, 1);
  }
}

// D/E, persistent: CTAs of 4 warps stream 4-line column tiles [pos][4] (swizzled, cp.async,
// the next tile in flight while the current one is transformed); warp g reads column g in the
// transform's spectral layout, runs the inverse 16 x 16 x 2 transform with a private exchange
// buffer and stores its cropped output row from registers (512 B per warp instruction).
constexpr int kR16CT = 4;
constexpr size_t r16_c2r_bytes(int T) { return (size_t(T) * 512 + size_t(512) * T + 4 * 32) * sizeof(double2); }

template <int MINB, int T = kR16CT>
__global__ void __launch_bounds__(T * 32, MINB) col_to_row_r16(WArgs a) {
  constexpr int L = 512;
  extern __shared__ double2 sm[];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const xb = sm + g * L;
  double2* const tile = sm + T * L;
  double2* const tws = tile + L * T;
  if (g == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) tws[32 * j + lane] = __ldg(a.tw + ((lane << j) & (L - 1)));
  }
  const unsigned ntiles_i = unsigned(a.n_inner + T - 1) / unsigned(T);
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto prefetch = [&](int64_t tix) {
    if (tix < ntiles) {
      const unsigned kq = unsigned(tix) / ntiles_i;
      const int i0 = int(unsigned(tix) - kq * ntiles_i) * T;
      const int lines_ok = min(T, a.n_inner - i0);
      const double2* base = a.in + int64_t(i0) * a.in_si + int64_t(kq) * a.in_sk;
      for (int e = threadIdx.x; e < a.in_nvalid * T; e += T * 32) {
        const int pos = e / T, t = e % T;
        cp_async16_zfill(&tile[mtile_at<T>(pos, t)], t < lines_ok ? base + t * a.in_si + pos * a.in_sp : a.in,
                         t < lines_ok);
      }
    }
    cp_async_commit();
  };
  const R16Tw<false> tw{tws, lane};
  const bool b = lane >= 16;
  const int k1 = lane & 15;
  int64_t tix = blockIdx.x;
  prefetch(tix);
  for (; tix < ntiles; tix += gridDim.x) {
    const unsigned kq = unsigned(tix) / ntiles_i;
    const int i0 = int(unsigned(tix) - kq * ntiles_i) * T;
    const bool ok = g < min(T, a.n_inner - i0);
    cp_async_wait0();
    __syncthreads();  // this tile's copies (issued by all threads) have landed
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int p = k1 + 16 * (i + 8 * int(b));
      v[i] = p < a.in_nvalid ? tile[mtile_at<T>(p, g)] : make_double2(0.0, 0.0);
      v[i + 8] = p + 256 < a.in_nvalid ? tile[mtile_at<T>(p + 256, g)] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // tile consumed by every warp
    prefetch(tix + gridDim.x);
    r16_r2_all<true>(v, b, std::make_integer_sequence<int, 8>{});
    dft16<true>(v);
#pragma unroll
    for (int h = 0; h < 16; ++h) xb[r16_ex(k1, 2 * h + int(b))] = v[h];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = xb[r16_ex(q, lane)];
    tw.apply<true>(v);
    dft16_half_out<true>(v);
    const int line = i0 + (ok ? g : 0);
    double2* orow = a.out + int64_t(line) * a.out_si + int64_t(kq) * a.out_sk;
    if (a.pm.n) {  // fused transpose: the row goes straight to the rank owning line (z)
      const int q = a.pm.owner(line);
      orow = a.pm.base[q] + (a.pm.off[q] + int64_t(line) * a.out_si + int64_t(kq) * a.pm.sk[q]);
    }
    if (ok) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int pos = lane + 32 * e;
        if (pos < a.out_nvalid) orow[pos] = (a.scale == 1.0) ? v[e] : cscale(v[e], a.scale);
      }
    }
    __syncwarp();  // exchange buffer read out before the next tile's writes
  }
  cp_async_wait0();
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

int launch_transpose_r16(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s) {
  static const int mask = [] {  // FUSG_R16_T bitmask: 1 passes A/B, 2 passes D/E (default both)
    const char* e = getenv("FUSG_R16_T");
    return e ? atoi(e) : 3;
  }();
  if (!(mask & (r2c ? 1 : 2))) return 0;
  if (r2c ? (2 * a.in_nvalid > 512 || a.in_sp != 1) : (2 * a.out_nvalid > 512 || a.out_sp != 1)) return 0;
  const int64_t tiles8 = int64_t((a.n_inner + 7) / 8) * a.n_outer;
  if (tiles8 >= (int64_t(1) << 31)) return 0;
  cudaError_t err;
  if (r2c) {
    const auto fn = warp_row_to_col_r16;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kR16TileBytes)) != cudaSuccess) {
      set_error(FUSG_CUDA, "transposing pass (16x16x2): cannot configure shared memory");
      return -1;
    }
    fn<<<unsigned(tiles8), 256, kR16TileBytes, s>>>(a);
  } else {
    // FUSG_R16_C2R_T: lines per tile (4: 3 CTAs of 4 warps per SM; 8: 128-byte tile segments,
    // one CTA of 8 warps per SM)
    static const int T = [] {
      const char* e = getenv("FUSG_R16_C2R_T");
      return (e && atoi(e) == 8) ? 8 : 4;
    }();
    const auto fn = T == 8 ? col_to_row_r16<1, 8> : col_to_row_r16<3, 4>;
    const size_t bytes = r16_c2r_bytes(T);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) != cudaSuccess) {
      set_error(FUSG_CUDA, "transposing pass (16x16x2): cannot configure shared memory");
      return -1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, T * 32, bytes) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      return 0;
    }
    const int64_t tiles = int64_t((a.n_inner + T - 1) / T) * a.n_outer;
    static const int waves = [] {  // FUSG_R16_C2R_WAVES: CTAs per SM slot (1 = persistent)
      const char* e = getenv("FUSG_R16_C2R_WAVES");
      return e ? std::max(1, atoi(e)) : 1;
    }();
    const int64_t grid = std::min<int64_t>(tiles, int64_t(per_sm) * ctx->num_sms * waves);
    fn<<<unsigned(grid), T * 32, bytes, s>>>(a);
  }
  ctx->launches++;
  err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "transposing pass (16x16x2)");
    return -1;
  }
  return 1;
}

int launch_ab_fused_r16(fusg_ctx* ctx, const ABFused& f, cudaStream_t s) {
  // FUSG_AB_FUSED=1 opts in.  Measured on cfg2: DRAM traffic of A+B drops from 2.3 to 1.33 GB
  // (the ring stays in L2, its dead lines discarded), but the launch takes 0.63 ms against
  // 0.434 ms for the two separate launches, so it is off by default.  The persistent item loop
  // itself is the cost: with every A item before every B item and the whole bufA as the ring
  // (FUSG_ABF_MODE=16, DRAM traffic as unfused) it also takes 0.63 ms; ncu shows CTA-barrier
  // and FP64-dependency stalls at 16 warps per SM where the one-shot launches overlap CTAs.
  static const bool on = [] {
    const char* e = getenv("FUSG_AB_FUSED");
    return e && atoi(e) != 0;
  }();
  if (!on) return 0;
  const auto fn = ab_fused_r16;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kABFusedBytes)) != cudaSuccess) {
    set_error(FUSG_CUDA, "fused passes A+B: cannot configure shared memory");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, kABFusedBytes) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  if (cudaMemsetAsync(f.sync, 0, sizeof(int) * (1 + 2 * size_t(f.slabs)), s) != cudaSuccess) {  // counters
    cuda_error(cudaGetLastError(), "fused passes A+B: reset");
    return -1;
  }
  static const int mode = [] {
    const char* e = getenv("FUSG_ABF_MODE");
    return e ? atoi(e) : 0;
  }();
  ABFused g = f;
  g.mode = mode;
  if (mode & 16) {  // experiment (Nz a multiple of 8): the whole bufA as the ring
    if (int64_t(g.slabs) * 8 != g.nz) return 0;
    g.ring = g.slabs;
  }
  fn<<<unsigned(per_sm * ctx->num_sms), 256, kABFusedBytes, s>>>(g);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "fused passes A+B");
    return -1;
  }
  return 1;
}

}  // namespace fusg
