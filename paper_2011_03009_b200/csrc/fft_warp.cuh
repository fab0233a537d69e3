// Warp-per-line Stockham FFT engine for the hot padded lengths (L <= 512).
//
// A line of L points is owned by LANES lanes of one warp (32 / LANES lines per warp); each
// lane holds E = L / LANES values in registers.  Stages exchange data through a shared-memory
// line buffer with __syncwarp only (no CTA barriers inside a transform).  The buffer is
// swizzled, addr(pos) = pos ^ ((pos >> 3) & 7) per 8-element row, which makes both Stockham
// access patterns (lane-consecutive reads, stride-R writes) bank-conflict-free.
//
// Twiddles: one table load w^k per butterfly and stage; the powers w^{rk}, r < R, come from a
// depth-3 multiply tree (<= 3 roundings; FUSG_TWIDDLE_TREE=0 selects successive multiplication,
// fewer live registers but measured slower), versus loading all R-1 from shared/L1.
//
// Stage s (radix R, NS = product of earlier radices, NB = L/R): butterfly j = lane + LANES*b,
// slot e = b*R + r holds position j + r*NB on input and (j - j%NS)*R + j%NS + r*NS on output.
#pragma once
#include "fft_static.cuh"

namespace fusg {

__device__ __forceinline__ int swz(int p) { return p ^ ((p >> 3) & 7); }

// w^r for r = 1..R-1 from w (compile-time R), INV -> conjugate handled by the caller
template <int R>
__device__ __forceinline__ void twiddle_powers(double2 w, double2* p) {
  p[1] = w;
  if constexpr (R > 2) p[2] = cmul(w, w);
  if constexpr (R > 3) p[3] = cmul(p[2], w);
  if constexpr (R > 4) p[4] = cmul(p[2], p[2]);
  if constexpr (R > 5) p[5] = cmul(p[4], w);
  if constexpr (R > 6) p[6] = cmul(p[3], p[3]);
  if constexpr (R > 7) p[7] = cmul(p[4], p[3]);
}

template <class RL, int LANES>
struct WarpGeom {
  static constexpr int L = RL::len();
  static constexpr int E = L / LANES;
  static_assert(L % LANES == 0, "line must split evenly over its lanes");
};

// Input slot positions of stage S for lane `lane`.
template <class RL, int LANES, int S>
__device__ __forceinline__ int in_pos(int lane, int e) {
  constexpr int R = RL::at(S);
  constexpr int NB = RL::len() / R;
  const int b = e / R, r = e % R;
  return lane + LANES * b + r * NB;
}

template <class RL, int LANES, int S>
__device__ __forceinline__ int out_pos(int lane, int e) {
  constexpr int R = RL::at(S);
  constexpr int NS = RL::ns(S);
  const int b = e / R, r = e % R;
  const int j = lane + LANES * b;
  const int k = j % NS;
  return (j - k) * R + k + r * NS;
}

// Twiddle source: one L1/global table load w^k per butterfly and stage, powers from a multiply
// tree.  (Keeping a persistent lane's twiddles in registers instead was measured slower: it
// pushes pass C past 255 registers.)
struct TwTable {
  const double2* tw;
  template <class RL, int LANES, int S, int R>
  __device__ __forceinline__ void powers(int lane, int b, double2* p) const {
    constexpr int NS = RL::ns(S);
    constexpr int TWS = RL::len() / (NS * R);
    const int k = (lane + LANES * b) % NS;
    twiddle_powers<R>(__ldg(tw + k * TWS), p);
  }
};

// Twiddle + butterflies of stage S on the register array v (input slots -> output slots).
// PRUNE bit 1: stage 0's inputs r >= R/2 are zero padding; bit 2: the last stage's outputs
// r >= R/2 are cropped (radix-8 stages use the pruned butterflies).
template <class RL, int LANES, bool INV, int S, int PRUNE, class Tw>
__device__ __forceinline__ void warp_stage_compute(double2* v, int lane, const Tw& tw) {
  constexpr int R = RL::at(S);
  constexpr int NS = RL::ns(S);
  constexpr int L = RL::len();
  constexpr int E = L / LANES;
  constexpr int B = E / R;
  static_assert(E % R == 0, "each lane must own whole butterflies");
  // (recomputing the powers per butterfly even when k repeats keeps fewer registers live:
  // sharing them across butterflies was measured slower in the register-bound pass C)
#pragma unroll
  for (int b = 0; b < B; ++b) {
    if constexpr (NS > 1) {
      double2 p[8];
      tw.template powers<RL, LANES, S, R>(lane, b, p);
#pragma unroll
      for (int r = 1; r < R; ++r) v[b * R + r] = INV ? cmulc(v[b * R + r], p[r]) : cmul(v[b * R + r], p[r]);
    }
    if constexpr (R == 8 && S == 0 && (PRUNE & 1)) dft8_half_in<INV>(v + b * R);
    else if constexpr (R == 8 && S == RL::n - 1 && (PRUNE & 2)) dft8_half_out<INV>(v + b * R);
    else dft<R, INV>(v + b * R);
  }
}

// Exchange barriers of a line: one warp (__syncwarp) or a lane group of several warps (a named
// barrier over exactly those warps' threads; ids 1..15, 0 is __syncthreads').
struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
template <int THREADS>
struct GroupSync {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(THREADS) : "memory"); }
};

// Full transform of the LANES-lane line owned by this lane group.
//   src.load(pos, e) feeds stage 0; dst.store(pos, e, v) receives the last stage's outputs.
//   ex.at(pos): this line's swizzled shared exchange slot for position pos.
template <class RL, int LANES, bool INV, int PRUNE = 0, int S = 0, class Ex, class Tw, class Src,
          class Dst, class Sync = WarpSync>
__device__ __forceinline__ void warp_fft(double2* v, Ex ex, int lane, const Tw& tw, Src& src, Dst& dst,
                                         Sync sync = Sync{}) {
  constexpr int E = RL::len() / LANES;
  constexpr int R0 = RL::at(0);
  if constexpr (S == 0) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((PRUNE & 1) && R0 == 8 && (e % R0) >= R0 / 2) continue;  // zero padding: not loaded
      v[e] = src.load(in_pos<RL, LANES, 0>(lane, e), e);
    }
  }
  warp_stage_compute<RL, LANES, INV, S, PRUNE>(v, lane, tw);
  if constexpr (S + 1 < RL::n) {
    sync();  // all lanes finished reading the buffer (previous stage / caller)
#pragma unroll
    for (int e = 0; e < E; ++e) ex.at(out_pos<RL, LANES, S>(lane, e)) = v[e];
    sync();
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = ex.at(in_pos<RL, LANES, S + 1>(lane, e));
    warp_fft<RL, LANES, INV, PRUNE, S + 1>(v, ex, lane, tw, src, dst, sync);
  } else {
    constexpr int RL_ = RL::at(S);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((PRUNE & 2) && RL_ == 8 && (e % RL_) >= RL_ / 2) continue;  // cropped: never stored
      dst.store(out_pos<RL, LANES, S>(lane, e), e, v[e]);
    }
  }
}

// ------------------------------------------------------------------ endpoints
// Column of a swizzled [pos][8] tile: element (pos, t) lives at pos*8 + (t ^ swz-bits).
__device__ __forceinline__ int tile_at(int pos, int t) { return pos * 8 + (t ^ ((pos ^ (pos >> 3)) & 7)); }

struct PrivEx {  // private line buffer of L elements
  double2* b;
  __device__ __forceinline__ double2& at(int pos) const { return b[swz(pos)]; }
};
struct TileEx {  // the line's own column of the [pos][8] tile (in-place exchange)
  double2* tile;
  int t;
  __device__ __forceinline__ double2& at(int pos) const { return tile[tile_at(pos, t)]; }
};

struct TileColIn {
  const double2* tile;
  int t, nvalid;
  __device__ __forceinline__ double2 load(int pos, int) const {
    return pos < nvalid ? tile[tile_at(pos, t)] : make_double2(0.0, 0.0);
  }
};
struct TileColOut {
  double2* tile;
  int t;
  __device__ __forceinline__ void store(int pos, int, double2 v) const { tile[tile_at(pos, t)] = v; }
};
struct RowIn {  // global line with position stride sp (1 for rows), zero beyond nvalid
  const double2* p;
  int64_t sp;
  int nvalid;
  bool ok;
  __device__ __forceinline__ double2 load(int pos, int) const {
    return (ok && pos < nvalid) ? __ldg(p + pos * sp) : make_double2(0.0, 0.0);
  }
};
struct RowOut {
  double2* p;
  int64_t sp;
  int nvalid;
  bool ok;
  double scale;
  __device__ __forceinline__ void store(int pos, int, double2 v) const {
    if (ok && pos < nvalid) p[pos * sp] = (scale == 1.0) ? v : cscale(v, scale);
  }
};
struct StagedRowIn {  // a line staged (swizzled) in shared memory by cp.async, zero beyond nvalid
  const double2* b;
  int nvalid;
  __device__ __forceinline__ double2 load(int pos, int) const {
    return pos < nvalid ? b[swz(pos)] : make_double2(0.0, 0.0);
  }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const size_t ga = __cvta_generic_to_global(gmem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(ga) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// 1-D bulk copies (TMA, cp.async.bulk) into shared memory with an mbarrier transaction count:
// one elected lane stages a whole contiguous row (full 128-byte smem lines, no per-lane
// LDGSTS), the consumers wait on the barrier's phase parity.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {  // inits visible to the async proxy
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Orders this thread's earlier generic-proxy shared-memory accesses -- and, through the
// barrier that precedes every refill, the other threads' reads of the buffer -- before the
// async-proxy (bulk copy) writes that follow.  Without it a refill could land while a lane's
// shared load of the old contents is still queued: measured on the B200 as rare bitwise
// differences between repeated applies (pass C at L = 256, one apply in ~10 at 224 x 224 lines).
__device__ __forceinline__ void refill_fence() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// stage `bytes` from src into dst (lane 0 of the caller's group issues; bytes > 0), after the
// buffer's previous contents were read by the generic proxy
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  refill_fence();
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, src, bytes, bar);
}

struct RegsOut {  // keep the last stage's outputs in the caller's registers
  double2* v;
  __device__ __forceinline__ void store(int, int e, double2 x) const { v[e] = x; }
};
struct RegsIn {
  const double2* v;
  __device__ __forceinline__ double2 load(int, int e) const { return v[e]; }
};

}  // namespace fusg
