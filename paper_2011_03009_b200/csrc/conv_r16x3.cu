// Pass C of the apply at padded z length 1536 = 3 x 512: one CTA of three warps per line, warp
// r owning the residue-r sub-transform, each a 16 x 16 x 2 warp transform (r16.cuh).
//
// Forward (decimation in frequency by 3; x[n] = 0 for n >= 768, the zero padding):
//   X[3k' + r] = DFT512_k'( y_r ),  y_r[m] = W1536^(m r) (x[m] + W3^r x[m + 512]),  m < 512
// (x[m + 1024] is padding).  The spectrum is multiplied by the folded K^ row in the warp's
// half-exchanged layout.  Inverse (decimation in time by 3, unnormalised, cropped to n < 768):
//   z_r = IDFT512( Z_r ),  t_r[n'] = W1536^(-n' r) z_r[n'],
//   x[n'] = t0 + t1 + t2,  x[n' + 512] = t0 + W3^-1 t1 + W3^-2 t2   (n' < 256).
// The per-lane part W1536^(lane r) of the input twiddle W1536^((32 n1 + lane) r) commutes with
// stage A's in-lane radix 16 and is merged into its twiddle (r16_twiddle_u); the per-slot part
// W48^(n1 r) is a warp-uniform table value.  The three t_r meet in shared memory and the CTA
// writes the cropped row with coalesced stores.
//
// Per line (three warps): one 12 KB bulk copy of the input row and one of the folded K^ row,
// both issued one line ahead; three shared exchanges plus shuffle half-exchanges per direction.
// Against the 64-lane radix (8, 8, 3, 8) kernel it keeps 16 values per lane (no spills at
// 4 CTAs = 12 warps per SM) and moves ~2000 instead of ~2800 shared wavefronts per line.
#include <algorithm>
#include <cstdlib>

#include "r16.cuh"
#include "tma.cuh"

namespace fusg {

#ifndef FUSG_X3_OROW
#define FUSG_X3_OROW 1  // pass C: the staging thread leaves each line's output-row offset in shared memory
#endif
#ifndef FUSG_X3_PAD
#define FUSG_X3_PAD 1  // pass C exchange buffers as 16 rows of 33 entries (0: XOR-swizzled [16][32])
#endif
// shared-memory layout (double2 offsets) of one CTA
template <int MODE = 1>
struct X3Smem {
  static constexpr bool STAGED = MODE != 0;
  static constexpr int XS = FUSG_X3_PAD ? 16 * 33 : 512;  // exchange buffer of one warp (X3W<.., PAD>)
  static constexpr int XB = 0;             // [3][XS] exchange buffers, then the t_r rows
  static constexpr int KB = 3 * XS;        // folded K^ row (769, padded to 770); MODE 2: also the input row
  static constexpr int TW = KB + 770;      // [4][32] W512^(lane 2^j)
  static constexpr int US = TW + 128;      // [3][32] W1536^(lane r)
  static constexpr int C48 = US + 96;      // [48] W48^j
  static constexpr int SB = MODE == 2 ? KB : C48 + 48;  // staged input row (<= 768 positions)
  static constexpr int END = C48 + 48 + (MODE == 1 ? 768 : 0);
  // + 2 mbarriers + 2 output-row offsets (MODE 1: thread 0 leaves the row offset of the line it
  // stages for the other threads, which then skip the line -> (ky, kx) divisions)
  static constexpr size_t BYTES = size_t(END) * sizeof(double2) + 4 * sizeof(uint64_t);
};

// W48^j = W1536^(32 j) in the constant bank (the same long-double values as the twiddle table):
// the residue-specialised slot twiddles below read them as constant operands, no shared loads
__constant__ double2 c_w48[48];
// W32^j = W1024^(32 j) for the 2 x 512 transposing passes
__constant__ double2 c_w32t[32];

// shared load the compiler may not hoist out of the line loop (keeps loop-invariant twiddles out
// of the register budget)
__device__ __forceinline__ double2 lds_fresh(const double2* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

// Per-warp pieces of the 1536 = 3 x 512 transform (warp r owns residue r).  SMEMTW: the lane
// twiddles W1536^(lane r), W512^(lane 2^j) are read from the CTA tables at each use instead of
// living in 20 registers for the whole kernel (the 5-CTA pass C needs <= 136 registers).
template <bool SMEMTW, int R = 3, bool PAD = false>
struct X3W {
  static_assert(R == 2 || R == 3, "lines of 2 x 512 or 3 x 512");
  // exchange buffer index of (row, col): XOR-swizzled [16][32], or (PAD) rows of 33 entries --
  // also conflict-free for both access patterns and affine in the lane, so every offset folds
  // into the instruction's immediate (the XOR costs a LOP3 per access, 5 % of pass C's instructions)
  static constexpr int XSTRIDE = PAD ? 16 * 33 : 512;
  static __device__ __forceinline__ int ex(int row, int col) { return PAD ? row * 33 + col : r16_ex(row, col); }
  double2 u, w1, w2, w4, w8;  // W1536^(lane r); W512^(lane 2^j) (registers: !SMEMTW)
  const double2* usp;         // &us[32 r + lane], &tws[lane] (SMEMTW)
  const double2* twp;
  const double2* c48;         // W48^j (shared)
  int r, k1;
  bool b;
  double c3, s3;              // W3^r = c3 + i s3
  __device__ __forceinline__ X3W(const double2* sm_us, const double2* tws, const double2* c48_, int r_, int lane)
      : c48(c48_), r(r_), k1(lane & 15), b(lane >= 16) {
    usp = sm_us + 32 * r + lane;
    twp = tws + lane;
    if constexpr (!SMEMTW) {
      u = *usp;
      w1 = twp[0];
      w2 = twp[32];
      w4 = twp[64];
      w8 = twp[96];
    }
    c3 = r == 0 ? 1.0 : -0.5;
    s3 = r == 0 ? 0.0 : r == 1 ? -0.8660254037844386467637 : 0.8660254037844386467637;
  }
  template <bool CONJ>
  __device__ __forceinline__ void twiddle_u(double2* v) const {
    if constexpr (SMEMTW) {
      r16_twiddle_u<CONJ>(v, lds_fresh(usp), lds_fresh(twp), lds_fresh(twp + 32), lds_fresh(twp + 64), lds_fresh(twp + 96));
    } else {
      r16_twiddle_u<CONJ>(v, u, w1, w2, w4, w8);
    }
  }
  // The three residues run the same instructions (residue 0 multiplies by exact ones), so the
  // warps of a CTA reach its barriers together.
  // y_r[32 n1 + lane] without its W1536 twiddle: x[m] + W3^r x[m + 512] (x zero beyond nv);
  // R = 2 (nv <= 512): x[m]
  __device__ __forceinline__ void gather(double2* v, const double2* row, int nv, int lane) const {
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) {
      const int m = 32 * n1 + lane;
      double2 x0 = m < nv ? row[m] : make_double2(0.0, 0.0);
      if (R == 3 && n1 < 8) {
        const double2 x1 = m + 512 < nv ? row[m + 512] : make_double2(0.0, 0.0);
        x0 = make_double2(fma(c3, x1.x, fma(-s3, x1.y, x0.x)), fma(c3, x1.y, fma(s3, x1.x, x0.y)));
      }
      v[n1] = x0;
    }
  }
  // forward: y_r (gathered) -> X[3k' + r] in the half-exchanged layout (slot i: k' = k1 + 16 (i + 8 b),
  // slot i + 8: k' + 256); xr: this warp's 512-entry exchange buffer
  __device__ __forceinline__ void forward(double2* v, double2* xr, int lane) const {
    forward_a(v);
    forward_b(v, xr, lane);
  }
  // stage A of the forward transform (registers only)
  __device__ __forceinline__ void forward_a(double2* v) const {
    slot_twiddle<false>(v);  // W48^(n1 r), n1 r < 48
    dft16<false>(v);
    twiddle_u<false>(v);
  }
  // the exchange, stage B, and the last radix 2 fused with the folded-K^ multiply: the two K^
  // values of step I + 1 are read from shared memory while step I shuffles, so their latency
  // hides behind the half-exchange (the separate multiply loop stalled on each load)
  __device__ __forceinline__ void forward_b_mulk(double2* v, double2* xr, int lane, const double2* kb,
                                                 uint64_t* kbar, unsigned kph) const {
#pragma unroll
    for (int k = 0; k < 16; ++k) xr[ex(k, lane)] = v[k];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = xr[ex(k1, 2 * h + int(b))];
    dft16<false>(v);
    mbar_wait(kbar, kph);  // this line's K^ row has landed
    // slot i holds X[3 k' + r] with k' = k1 + 16 (i + 8 b) (< 256) and slot i + 8 its k' + 256 twin,
    // whose folded K^ index is 768 - j
    r16_fwd_r2_mulk_all<48, 768>(v, b, kb, 3 * k1 + 384 * int(b) + r, std::make_integer_sequence<int, 8>{});
  }
  // the exchange through xr and stage B
  __device__ __forceinline__ void forward_b(double2* v, double2* xr, int lane) const {
#pragma unroll
    for (int k = 0; k < 16; ++k) xr[ex(k, lane)] = v[k];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = xr[ex(k1, 2 * h + int(b))];
    dft16<false>(v);
    r16_r2_all<false>(v, b, std::make_integer_sequence<int, 8>{});
  }
  // inverse: Z_r (half-exchanged layout) -> t_r[n'] = W1536^(-n' r) z_r[n'] in the natural
  // layout (slot n1 = position 32 n1 + lane)
  __device__ __forceinline__ void inverse(double2* v, double2* xr, int lane) const {
    r16_r2_all<true>(v, b, std::make_integer_sequence<int, 8>{});
    dft16<true>(v);
#pragma unroll
    for (int h = 0; h < 16; ++h) xr[ex(k1, 2 * h + int(b))] = v[h];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xr[ex(k, lane)];
    twiddle_u<true>(v);
    dft16<true>(v);
    slot_twiddle<true>(v);
  }
  // v[n1] *= W48^(n1 r) (CONJ: its conjugate); residue 0 multiplies by ones and skips it
  template <bool CONJ>
  __device__ __forceinline__ void slot_twiddle(double2* v) const {
    auto m = [](double2 x, double2 t) { return CONJ ? cmulc(x, t) : cmul(x, t); };
    if constexpr (R == 2) {  // W32^(n1 r)
      if (r == 1) {
#pragma unroll
        for (int n1 = 1; n1 < 16; ++n1) v[n1] = m(v[n1], c_w32t[n1]);
      }
      return;
    }
    if (r == 1) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = m(v[n1], c_w48[n1]);
    } else if (r == 2) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = m(v[n1], c_w48[2 * n1]);
    }
  }
};
using X3Warp = X3W<false>;

// cropped row from the three t_r rows: x[n'] = t0 + t1 + t2, x[n' + 512] = t0 + W3^-1 t1 + W3^-2 t2
// SCALED = false: the caller knows sc == 1 (pass C always; the per-element test-and-select costs
// issue slots)
template <bool SCALED = true>
__device__ __forceinline__ void x3_recombine(const double2* t0r, const double2* t1r, const double2* t2r, int n,
                                             int onv, double sc, double2* out) {
  constexpr double kS3 = 0.8660254037844386467637;
  const double2 t0 = t0r[n], t1 = t1r[n], t2 = t2r[n];
  const double2 s = cadd(t1, t2);
  if (n < onv) {
    const double2 o = cadd(t0, s);
    out[n] = (!SCALED || sc == 1.0) ? o : cscale(o, sc);
  }
  if (n + 512 < onv) {
    const double2 d = csub(t1, t2);
    const double2 o = make_double2(t0.x - 0.5 * s.x - kS3 * d.y, t0.y - 0.5 * s.y + kS3 * d.x);
    out[n + 512] = (!SCALED || sc == 1.0) ? o : cscale(o, sc);
  }
}

// the per-CTA twiddle tables: tws [4][32] W512^(lane 2^j), us [3][32] W1536^(lane r), c48 [48]
template <int R = 3>
__device__ __forceinline__ void x3_tables(const double2* twL, double2* tws, double2* us, double2* c48) {
  constexpr int L = 512 * R;  // twL: the W_L table; tws = W512^(lane 2^j), us = W_L^(lane r), c48 = W_L^(32 j)
  for (int e = threadIdx.x; e < 128; e += blockDim.x) tws[e] = __ldg(twL + (((R * (e & 31)) << (e >> 5)) % L));
  for (int e = threadIdx.x; e < 32 * R; e += blockDim.x) us[e] = __ldg(twL + (e & 31) * (e >> 5));
  for (int e = threadIdx.x; e < 16 * R; e += blockDim.x) c48[e] = __ldg(twL + 32 * e);
}

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ---------------------------------------------------------------------------- pass C
// CTA of three warps, persistent over lines; the input and K^ rows are staged by 1-D bulk
// copies one line ahead (the refill is issued after a CTA barrier: measured faster than
// letting the warps drift apart with last-arriver refills or producer / consumer barriers,
// 29.8 vs 32.8-33.6 ms at cfg5).
// STAGED = false: the input row is read straight from global memory (prefetched into L2 one
// line ahead), which frees 12 KB per CTA for a fifth CTA (15 warps) per SM.
#ifndef FUSG_X3_MINB
#define FUSG_X3_MINB 4  // CTAs per SM the staged pass C's register budget targets (4: <= 168 registers)
#endif
// MODE 1 (default): input row and K^ row in their own buffers, each refilled one line ahead.
// MODE 2: one staging buffer holds the input row until the gather, then this line's K^ row
// (loaded while the forward transform runs), then the next input row (loaded during the inverse
// and the recombination); 41 KB of shared memory and lane twiddles read from the tables let 5
// CTAs (15 warps) share an SM. MODE 0: input rows read from L2 (5 CTAs).
// FULL: every row holds 768 valid inputs and outputs (cfg5): the bounds are compile-time, so the
// gather and the recombination carry no predicates or zero fills.
template <int MODE, bool FULL = false>
__global__ void __launch_bounds__(96, MODE == 1 ? FUSG_X3_MINB : 5) conv_r16x3(WArgs a) {
  constexpr bool STAGED = MODE != 0;
  constexpr int HZ = 769;
  using X3Smem = fusg::X3Smem<MODE>;
  extern __shared__ double2 sm[];
  const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const xb = sm + X3Smem::XB;
  double2* const xr = xb + X3Smem::XS * r;
  double2* const sb = sm + X3Smem::SB;
  double2* const kb = sm + X3Smem::KB;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + X3Smem::END);
  x3_tables(a.tw, sm + X3Smem::TW, sm + X3Smem::US, sm + X3Smem::C48);
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const X3W<MODE == 2, 3, FUSG_X3_PAD != 0> W(sm + X3Smem::US, sm + X3Smem::TW, sm + X3Smem::C48, r, lane);
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t stride = gridDim.x;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) {  // line < 2^31 (host-checked)
    conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx);
  };
  int64_t* const orow = reinterpret_cast<int64_t*>(bars + 2);  // [2] output-row offsets by line parity
  auto prefetch_in = [&](int64_t line, unsigned slot) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      const double2* src = a.in + ky * a.in_si + int64_t(kx) * a.in_sk;
      if constexpr (MODE == 1 && FUSG_X3_OROW) orow[slot] = ky * a.out_si + int64_t(kx) * a.out_sk;
      if constexpr (STAGED) {
        bulk_stage(sb, src, unsigned(a.in_nvalid) * sizeof(double2), bars);
      } else {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(unsigned(a.in_nvalid) * 16u)
                     : "memory");
      }
    }
  };
  auto prefetch_k = [&](int64_t line) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      bulk_stage(kb, a.ko.line(ky, kx), HZ * sizeof(double2), bars + 1);
    }
  };
  const int nv = FULL ? 768 : a.in_nvalid, onv = FULL ? 768 : a.out_nvalid;
  int64_t line = blockIdx.x;
  if (threadIdx.x == 0) {
    prefetch_in(line, 0);
    if constexpr (MODE != 2) prefetch_k(line);
  }
  unsigned ph = 0;  // both staging barriers complete once per line
  for (; line < nlines; line += stride, ph ^= 1) {
    double2 v[16];
    if constexpr (STAGED) {
      mbar_wait(bars, ph);
      W.gather(v, sb, nv, lane);
    } else {
      int ky, kx;
      coords(line, ky, kx);
      W.gather(v, a.in + ky * a.in_si + int64_t(kx) * a.in_sk, nv, lane);
    }
    __syncthreads();  // the staged row is read by all three warps: refill it
    if (threadIdx.x == 0) {
      if constexpr (MODE == 2) prefetch_k(line);  // this line's K^ row into the same buffer
      else prefetch_in(line + stride, ph ^ 1u);
    }
    // X[3k' + r] times the folded K^ row, fused into the last forward stage
    W.forward_a(v);
    W.forward_b_mulk(v, xr, lane, kb, bars + 1, ph);
    __syncthreads();  // K^ row read
    if (threadIdx.x == 0) {
      if constexpr (MODE == 2) prefetch_in(line + stride, ph ^ 1u);
      else prefetch_k(line + stride);
    }
    W.inverse(v, xr, lane);
    __syncwarp();  // every lane has read its exchange slots
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) xr[32 * n1 + lane] = v[n1];
    __syncthreads();
    double2* out;
    if constexpr (MODE == 1 && FUSG_X3_OROW) {
      out = a.out + orow[ph];  // left by thread 0 when it staged this line (barriers in between)
    } else {
      int ky, kx;
      coords(line, ky, kx);
      out = a.out + ky * a.out_si + int64_t(kx) * a.out_sk;
    }
    if (a.scale == 1.0) {  // (always, from the apply: the scale rides on pass E)
      for (int n = threadIdx.x; n < 512; n += 96) x3_recombine<false>(xb, xb + X3Smem::XS, xb + 2 * X3Smem::XS, n, onv, 1.0, out);
    } else {
      for (int n = threadIdx.x; n < 512; n += 96) x3_recombine(xb, xb + X3Smem::XS, xb + 2 * X3Smem::XS, n, onv, a.scale, out);
    }
    // (the next line's staging barrier orders these reads before its exchange writes)
  }
}

// ---------------------------------------------------------------------------- pass C, quad CTA + TMEM
// One CTA of twelve warps per SM runs the (up to) four lines (+-ky, +-kx) that read one folded
// K^ row: warp 4 r + j owns residue r of line j.  The three warps of a line sit in the same
// tensor-memory lane quarter (warp index mod 4 = j) and lane l of each holds position
// 32 n1 + l of its t_r, so the recombination x[n'] = t0 + t1 + t2 is lane-local: every warp
// parks its t_r in tensor memory (tcgen05.st, 64 columns), and after a 96-thread named barrier
// reads back the slots it combines (tcgen05.ld) and stores them -- no shared-memory round trip
// (384 of ~2290 LSU wavefronts per line), on a data path separate from the shared-memory pipe
// (tools/mb/tmem_ldst.cu: >= 184 B/clk/SM written, >= 236 B/clk/SM read with 12 warps).
// The K^ row is staged once per CTA (three buffers, two rows ahead; each warp arrives on the
// buffer's "read" mbarrier and thread 0 waits on it before the refill, so no CTA-wide barrier
// runs in the loop); each line's input row is staged per line group one row ahead.
// Measured (cfg5, B200): 30.5 ms against 29.4 ms for the three-warp kernel -- the lane twiddles
// have to come from the shared tables to stay under 168 registers (+120 wavefronts per line),
// the three warps of a line share one scheduler (their lane quarter) and hit the FP64 pipe
// together, and neither a CTA barrier taken at staggered points (38.1 ms) nor mbarriers waited
// on late with t_r double-buffered (31.7 ms) helped.  Opt-in: FUSG_X3_QUADTM=1.
struct X3QSmem {
  static constexpr int XB = 0;              // [12][512] exchange buffers, one per warp
  static constexpr int KB = 12 * 512;       // [3][770] folded K^ rows
  static constexpr int SB = KB + 3 * 770;   // [4][768] staged input rows, one per line
  static constexpr int TW = SB + 4 * 768;   // [4][32] W512^(lane 2^j)
  static constexpr int US = TW + 128;       // [3][32] W1536^(lane r)
  static constexpr int C48 = US + 96;       // [48]
  static constexpr int END = C48 + 48;
  // + 3 + 3 K^ barriers (landed / read), 4 row barriers, the tensor-memory base address
  static constexpr size_t BYTES = size_t(END) * sizeof(double2) + 11 * sizeof(uint64_t);
};

// 4 complex128 values of this lane -> 16 tensor-memory columns at taddr (four of them park a
// t_r: one 64-column store needs 64 consecutive registers, which made the allocator spill)
__device__ __forceinline__ void tm_st_c4(uint32_t taddr, const double2* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(__double2loint(v[0].x)), "r"(__double2hiint(v[0].x)), "r"(__double2loint(v[0].y)), "r"(__double2hiint(v[0].y)),
      "r"(__double2loint(v[1].x)), "r"(__double2hiint(v[1].x)), "r"(__double2loint(v[1].y)), "r"(__double2hiint(v[1].y)),
      "r"(__double2loint(v[2].x)), "r"(__double2hiint(v[2].x)), "r"(__double2loint(v[2].y)), "r"(__double2hiint(v[2].y)),
      "r"(__double2loint(v[3].x)), "r"(__double2hiint(v[3].x)), "r"(__double2loint(v[3].y)), "r"(__double2hiint(v[3].y))
      : "memory");
}
__device__ __forceinline__ void tm_st_c16(uint32_t taddr, const double2* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) tm_st_c4(taddr + 16u * unsigned(i), v + 4 * i);
}
// 4 complex128 values (16 columns) of this lane from taddr
__device__ __forceinline__ void tm_ld_c4(uint32_t taddr, double2* v) {
  uint32_t w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = make_double2(__hiloint2double(int(w[4 * i + 1]), int(w[4 * i])), __hiloint2double(int(w[4 * i + 3]), int(w[4 * i + 2])));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// x[n'] = t0 + t1 + t2 and x[n' + 512] = t0 + W3^-1 t1 + W3^-2 t2 (the expressions of x3_recombine)
__device__ __forceinline__ void x3_combine(double2 t0, double2 t1, double2 t2, double2& lo, double2& hi) {
  constexpr double kS3 = 0.8660254037844386467637;
  const double2 s = cadd(t1, t2), d = csub(t1, t2);
  lo = cadd(t0, s);
  hi = make_double2(t0.x - 0.5 * s.x - kS3 * d.y, t0.y - 0.5 * s.y + kS3 * d.x);
}

#ifndef FUSG_X3Q_SMEMTW
#define FUSG_X3Q_SMEMTW 1
#endif
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__global__ void __launch_bounds__(384, 1) conv_r16x3q(WArgs a) {
  constexpr int HZ = 769;
  extern __shared__ double2 sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = wid & 3, r = wid >> 2;  // line of the quad (tensor-memory lane quarter), residue
  double2* const xr = sm + X3QSmem::XB + 512 * wid;
  double2* const xs = sm + X3QSmem::SB + 768 * j;
  uint64_t* const kfull = reinterpret_cast<uint64_t*>(sm + X3QSmem::END);  // [3] K^ row landed
  uint64_t* const kfree = kfull + 3;                                        // [3] K^ row read by the 12 warps
  uint64_t* const xbar = kfull + 6 + j;
  uint32_t* const tm_slot = reinterpret_cast<uint32_t*>(kfull + 10);
  x3_tables(a.tw, sm + X3QSmem::TW, sm + X3QSmem::US, sm + X3QSmem::C48);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(kfull + i, 1);
    for (int i = 0; i < 3; ++i) mbar_init(kfree + i, 12);
    for (int i = 0; i < 4; ++i) mbar_init(kfull + 6 + i, 1);
    mbar_init_fence();
  }
  if (wid == 0) {  // 256 columns: t_r at columns 64 r (192 used)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tm_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tm_fence_before_sync();
  __syncthreads();
  tm_fence_after_sync();
  const uint32_t tm_base = *tm_slot;
  const uint32_t tm_lane = tm_base + (uint32_t(32 * j) << 16);
  const int Py = a.ko.Py, Px = a.ko.Px;
  const int Hy = Py / 2 + 1, Hx = Px / 2 + 1;
  const int nrows = Hy * Hx;  // folded K^ rows (< 2^31, host-checked)
  const int stride = int(gridDim.x);
  const int nv = a.in_nvalid, onv = a.out_nvalid;
  // line j of folded row q = fx Hy + fy: ky = fy or Py - fy (odd j), kx = fx or Px - fx (j >= 2);
  // false when that mirror is the line itself
  auto line_of = [&](int q, int& ky, int& kx) {
    const int fx = q / Hy, fy = q - fx * Hy;
    ky = fy, kx = fx;
    bool on = true;
    if (j & 1) {
      ky = Py - fy;
      on = fy > 0 && ky != fy;
    }
    if (j & 2) {
      kx = Px - fx;
      on = on && fx > 0 && kx != fx;
    }
    return on;
  };
  auto stage_k = [&](int q, int buf) {  // thread 0
    if (q < nrows) {
      const int fx = q / Hy, fy = q - fx * Hy;
      bulk_stage(sm + X3QSmem::KB + 770 * buf, a.ko.line(fy, fx), HZ * sizeof(double2), kfull + buf);
    }
  };
  auto stage_row = [&](int q) {  // residue 0, lane 0 of the line group, after the group's reads
    int ky, kx;
    if (q < nrows && line_of(q, ky, kx))
      bulk_stage(xs, a.in + ky * a.in_si + int64_t(kx) * a.in_sk, unsigned(nv) * sizeof(double2), xbar);
  };
  int q = int(blockIdx.x);
  if (threadIdx.x == 0) {
    stage_k(q, 0);
    stage_k(q + stride, 1);
  }
  if (r == 0 && lane == 0) stage_row(q);
  unsigned xph = 0;
#pragma unroll 1
  for (unsigned it = 0; q < nrows; q += stride, ++it) {
    const int buf = int(it % 3u);
    const double2* kb = sm + X3QSmem::KB + 770 * buf;
    int ky, kx;
    if (!line_of(q, ky, kx)) {  // the row's mirror line is the line itself: nothing to do
      if (lane == 0) {
        if (r == 0) stage_row(q + stride);
        // wait for the row like a working warp: an idle warp running ahead would arrive on this
        // buffer's next phase before the others have finished this one
        mbar_wait(kfull + buf, (it / 3u) & 1u);
        mbar_arrive(kfree + buf);
      }
      __syncwarp();
      continue;
    }
    // lane-derived shared-memory addresses are rebuilt every row instead of living in (spilled)
    // registers across the loop
    int ln = lane;
    asm volatile("" : "+r"(ln));
    const X3W<FUSG_X3Q_SMEMTW != 0> W(sm + X3QSmem::US, sm + X3QSmem::TW, sm + X3QSmem::C48, r, ln);
    double2 v[16];
    mbar_wait(xbar, xph);  // this line's row has landed
    xph ^= 1u;
    W.gather(v, xs, nv, ln);
    nbar_sync(1 + j, 96);  // the staged row is read by the line's three warps: refill it
    if (r == 0 && lane == 0) stage_row(q + stride);
    W.forward_a(v);
    W.forward_b_mulk(v, xr, ln, kb, kfull + buf, (it / 3u) & 1u);
    __syncwarp();
    if (lane == 0) mbar_arrive(kfree + buf);  // this warp has read the K^ row
    if (threadIdx.x == 0 && q + 2 * stride < nrows) {
      // the buffer of the previous row takes the row two ahead once all twelve warps have read it
      // (line 0 is never its own mirror, so this thread runs every row)
      const unsigned pb = (it + 2u) % 3u;
      if (it > 0) mbar_wait(kfree + pb, ((it - 1u) / 3u) & 1u);
      stage_k(q + 2 * stride, int(pb));
    }
    W.inverse(v, xr, ln);
    __syncwarp();  // every lane has read its exchange slots
    tm_st_c16(tm_lane + 64u * unsigned(r), v);
    tm_wait_st();
    tm_fence_before_sync();
    nbar_sync(1 + j, 96);  // the three t_r are in tensor memory
    tm_fence_after_sync();
    // warp r combines slots 4 r .. 4 r + 3 (r < 2: x[n'] and x[n' + 512]) or 8 .. 15 (x[n'] only)
    double2* out = a.out + ky * a.out_si + int64_t(kx) * a.out_sk;
    const double sc = a.scale;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && r < 2) break;
      const int s0 = r < 2 ? 4 * r : 8 + 4 * h;
      double2 t0[4], t1[4], t2[4];
      tm_ld_c4(tm_lane + 4u * unsigned(s0), t0);
      tm_ld_c4(tm_lane + 64u + 4u * unsigned(s0), t1);
      tm_ld_c4(tm_lane + 128u + 4u * unsigned(s0), t2);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2 lo, hi;
        x3_combine(t0[i], t1[i], t2[i], lo, hi);
        const int m = 32 * (s0 + i) + ln;
        if (m < onv) out[m] = sc == 1.0 ? lo : cscale(lo, sc);
        if (r < 2 && m + 512 < onv) out[m + 512] = sc == 1.0 ? hi : cscale(hi, sc);
      }
    }
    tm_fence_before_sync();  // these reads are ordered before the next row's tcgen05.st by its first group barrier
  }
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tm_base) : "memory");
}

// ---------------------------------------------------------------------------- passes A / B
// Row -> column (forward, pruned input <= 768 of 1536): a CTA of 3T warps transforms T adjacent
// lines (warp 3t + r: line t, residue r).  The T input rows (contiguous when the rows are
// dense) arrive by 1-D bulk copy one tile ahead; the spectra meet in a swizzled [pos][T] tile
// that aliases the twelve exchange buffers; the CTA stores 64-byte segments of T adjacent lines.
// FUSG_X3T_PAD bit 1: passes A / B (row -> column), bit 2: passes D / E.  Same-box A/B at cfg5:
// D / E 8.55 / 4.23 -> 8.41 / 4.16 ms padded, A / B 4.25 / 8.45 -> 4.30 / 8.57 ms, so only D / E.
#ifndef FUSG_X3T_PAD
#define FUSG_X3T_PAD 2
#endif
template <int T, int R = 3, bool PAD = false>
struct X3TSmem {
  static constexpr int L = 512 * R, H = 256 * R;
  // PAD: the warps' exchange buffers as 16 rows of 33 entries (X3W<.., PAD>) instead of the
  // XOR-swizzled [16][32]; the R T buffers then need a little more than the [L][T] tile they alias
  // (R = 3, T = 4: 6336 entries = 99 KB, still 1024-byte aligned for the second TMA tile)
  static constexpr int XS = PAD ? 16 * 33 : 512;
  static constexpr int TILE = L * T > R * T * XS ? L * T : R * T * XS;
  static constexpr int AREA = 0;            // [L][T] tile = R T exchange buffers
  static constexpr int STAGE = TILE;        // [T][L/2] staged input rows (r2c)
  static constexpr int TW = STAGE + H * T;  // tables as in X3Smem
  static constexpr int US = TW + 128;
  static constexpr int C48 = US + 32 * R;
  static constexpr int END = C48 + 16 * R;
  static constexpr size_t BYTES = size_t(END) * sizeof(double2) + sizeof(uint64_t);
  // TMA r2c: a second staging buffer after the tables (input rows two tiles ahead), 2 mbarriers
  static constexpr int STAGE2 = END;
  static constexpr size_t BYTES2 = size_t(STAGE2 + H * T) * sizeof(double2) + 2 * sizeof(uint64_t);
  // c2r: two [L][T] tiles (double-buffered), then the tables
  static constexpr int C_TW = 2 * TILE;
  static constexpr int C_US = C_TW + 128;
  static constexpr int C_C48 = C_US + 32 * R;
  static constexpr int C_END = C_C48 + 16 * R;
  static constexpr size_t C_BYTES = size_t(C_END) * sizeof(double2) + 2 * sizeof(uint64_t);
};

template <int T, int R = 3>
using X3TSmemA = X3TSmem<T, R, (FUSG_X3T_PAD & 1) != 0>;  // passes A / B
template <int T, int R = 3>
using X3TSmemD = X3TSmem<T, R, (FUSG_X3T_PAD & 2) != 0>;  // passes D / E

// CTAs per SM the transposing kernels' register budget targets: 1 per SM at T = 4 for 1536
// (12 warps, <= 168 registers); R = 2 (1024): 1 CTA (8 warps, ~200 registers), or with
// FUSG_X2T_MINB2 set at compile time a 128-register budget with the lane twiddles read from the
// CTA tables (no spills) -- but the double-buffered tiles (~130 KB) still allow one CTA per SM,
// so it only adds shared loads
#ifndef FUSG_X2T_MINB2
#define FUSG_X2T_MINB2 0
#endif
#define X3T_MINB ((T == 4 && R == 2 && FUSG_X2T_MINB2) ? 2 : 4 / T)
#define X3T_SMEMTW (T == 4 && R == 2 && FUSG_X2T_MINB2)  // lane twiddles from the CTA tables

// TMA (T = 4): the finished tile leaves by tensor-map box stores issued by one thread, and the
// next tile's stage-A arithmetic overlaps them; the area is rewritten (first exchange) only after
// the stores have read it.
// FULL: every row holds L / 2 valid inputs (no predicates or zero fills in the gather)
template <int T, bool TMA, int R = 3, bool FULL = false>
__global__ void __launch_bounds__(32 * R * T, X3T_MINB) r16x3_row_to_col(WArgs a, const __grid_constant__ CUtensorMap tm) {
  constexpr bool PAD = (FUSG_X3T_PAD & 1) != 0;
  using X3TSmem = fusg::X3TSmem<T, R, PAD>;
  constexpr int H = X3TSmem::H;  // L / 2
  extern __shared__ __align__(1024) double2 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = w % R, t = w / R;
  double2* const area = sm + X3TSmem::AREA;
  double2* const xr = area + X3TSmem::XS * w;
  // TMA: two staging buffers, filled two tiles ahead (the rows of pass B lie a z-plane apart and
  // arrive late one tile ahead); else one
  constexpr int NST = TMA ? 2 : 1;
  // (addressed arithmetically from the shared base: a runtime-indexed pointer array turns the
  // gather's shared loads into generic LD)
#ifndef FUSG_X3T_STAGEPTR
#define FUSG_X3T_STAGEPTR 0
#endif
#if FUSG_X3T_STAGEPTR
  double2* const stages_[2] = {sm + X3TSmem::STAGE, sm + X3TSmem::STAGE2};
  auto stage_of = [&](int sb) { return stages_[sb]; };
#else
  auto stage_of = [&](int sb) { return sm + (sb ? X3TSmem::STAGE2 : X3TSmem::STAGE); };
#endif
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + (TMA ? X3TSmem::STAGE2 + H * T : X3TSmem::END));
  x3_tables<R>(a.tw, sm + X3TSmem::TW, sm + X3TSmem::US, sm + X3TSmem::C48);
  if (threadIdx.x == 0) {
    for (int b = 0; b < NST; ++b) mbar_init(bars + b, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const X3W<X3T_SMEMTW, R, PAD> W(sm + X3TSmem::US, sm + X3TSmem::TW, sm + X3TSmem::C48, r, lane);
  const int nv = FULL ? H : a.in_nvalid;
  const int ntiles_i = (a.n_inner + T - 1) / T;
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto prefetch = [&](int64_t tix, int sb) {  // thread 0
    if (tix < ntiles) {
      const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
      const int k = int(unsigned(tix) / unsigned(ntiles_i));
      const int lines_ok = min(T, a.n_inner - i0);
      const double2* src = a.in + int64_t(i0) * a.in_si + int64_t(k) * a.in_sk;
      const unsigned row = unsigned(nv) * sizeof(double2);
      refill_fence();
      mbar_expect_tx(bars + sb, row * lines_ok);
      for (int tt = 0; tt < lines_ok; ++tt) bulk_g2s(stage_of(sb) + tt * H, src + tt * a.in_si, row, bars + sb);
    }
  };
  int64_t tix = blockIdx.x;
  if (threadIdx.x == 0)
    for (int b = 0; b < NST; ++b) prefetch(tix + int64_t(b) * gridDim.x, b);
  unsigned phs = 0;  // parity bit per staging buffer
  for (int it = 0; tix < ntiles; tix += gridDim.x, ++it) {
    const int sb = NST == 2 ? (it & 1) : 0;
    const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
    const int k = int(unsigned(tix) / unsigned(ntiles_i));
    const int lines_ok = min(T, a.n_inner - i0);
    mbar_wait(bars + sb, (phs >> sb) & 1u);
    phs ^= 1u << sb;
    double2 v[16];
    W.gather(v, stage_of(sb) + (t < lines_ok ? t : 0) * H, nv, lane);
    if constexpr (TMA) {
      W.forward_a(v);
      if (threadIdx.x == 0) bulk_wait_read0();  // the previous tile's box stores have read the area
    }
    __syncthreads();  // stage read by every warp: refill it with a later tile's rows
    if (threadIdx.x == 0) prefetch(tix + int64_t(NST) * gridDim.x, sb);
    if constexpr (TMA) {
      W.forward_b(v, xr, lane);
    } else {
      W.forward(v, xr, lane);
    }
    __syncthreads();  // every exchange buffer is read out: the area becomes the tile
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int p = R * (W.k1 + 16 * (i + 8 * int(W.b))) + r;
      area[mtile_at<T>(p, t)] = v[i];
      area[mtile_at<T>(p + H, t)] = v[i + 8];
    }
    __syncthreads();  // all T spectra are in the tile
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        smem_to_async_fence();
        for (int p0 = 0; p0 < a.out_nvalid; p0 += 256) tma_store_tile_box(&tm, area + p0 * T, 2 * i0, p0, k);
        bulk_commit();
      }
      continue;
    }
    double2* const base = a.out + int64_t(i0) * a.out_si + int64_t(k) * a.out_sk;
#pragma unroll 4
    for (int e = threadIdx.x; e < a.out_nvalid * T; e += 32 * R * T) {
      const int pos = e / T, tt = e % T;
      if (tt < lines_ok) {
        const double2 x = area[mtile_at<T>(pos, tt)];
        const double2 y = (a.scale == 1.0) ? x : cscale(x, a.scale);
        if (a.pm.n == 0) {
          base[tt * a.out_si + pos * a.out_sp] = y;
        } else {  // fused transpose: the segment goes straight to the rank owning it
          const int q = a.pm.owner(a.pm.by_pos ? pos : i0 + tt);
          a.pm.base[q][a.pm.off[q] + int64_t(i0 + tt) * a.out_si + int64_t(k) * a.pm.sk[q] + int64_t(pos) * a.out_sp] = y;
        }
      }
    }
    // (the next tile's staging barrier orders these reads before its exchange writes)
  }
  if constexpr (TMA) {
    if (threadIdx.x == 0) bulk_wait0();  // the last tile's stores complete before the CTA exits
  }
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

// ---------------------------------------------------------------------------- passes D / E
// Column -> row (inverse, cropped output <= 768): a CTA of 3T warps; the [pos][T] column tiles
// are double-buffered and filled by cp.async one tile ahead; each warp reads its residue's
// spectrum from the tile, the exchanges and the t_r rows reuse the current tile, and the CTA
// writes the T cropped rows with coalesced stores.
// TMA (T = 4): each column tile arrives by tensor-map box loads (one thread, one mbarrier per
// buffer) instead of per-thread cp.async; positions and lines beyond the field are zero-filled.
// FULL: full spectra in (L positions), L / 2 valid outputs per row
template <int T, bool TMA, int R = 3, bool FULL = false>
__global__ void __launch_bounds__(32 * R * T, X3T_MINB) r16x3_col_to_row(WArgs a, const __grid_constant__ CUtensorMap tm) {
  constexpr bool PAD = (FUSG_X3T_PAD & 2) != 0;
  using X3TSmem = fusg::X3TSmem<T, R, PAD>;
  constexpr int H = X3TSmem::H;
  constexpr int NT = 32 * R * T;
  extern __shared__ __align__(1024) double2 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = w % R, t = w / R;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + X3TSmem::C_END);  // [2], TMA only
  x3_tables<R>(a.tw, sm + X3TSmem::C_TW, sm + X3TSmem::C_US, sm + X3TSmem::C_C48);
  if (TMA && threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const X3W<X3T_SMEMTW, R, PAD> W(sm + X3TSmem::C_US, sm + X3TSmem::C_TW, sm + X3TSmem::C_C48, r, lane);
  const int ntiles_i = (a.n_inner + T - 1) / T;
  const int64_t ntiles = int64_t(ntiles_i) * a.n_outer;
  auto prefetch = [&](int64_t tix, double2* tile) {
    if constexpr (TMA) {
      if (tix < ntiles && threadIdx.x == 0) {
        const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
        const int k = int(unsigned(tix) / unsigned(ntiles_i));
        uint64_t* const bar = bars + (tile == sm ? 0 : 1);
        const int nbox = (a.in_nvalid + 255) / 256;
        refill_fence();
        mbar_expect_tx(bar, unsigned(nbox) * 256u * T * 16u);
        for (int b = 0; b < nbox; ++b) tma_load_tile_box(&tm, tile + b * 256 * T, bar, 2 * i0, 256 * b, k);
      }
      return;
    }
    if (tix < ntiles) {
      const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
      const int k = int(unsigned(tix) / unsigned(ntiles_i));
      const int lines_ok = min(T, a.n_inner - i0);
      const double2* base = a.in + int64_t(i0) * a.in_si + int64_t(k) * a.in_sk;
      for (int e = threadIdx.x; e < a.in_nvalid * T; e += NT) {
        const int pos = e / T, tt = e % T;
        cp_async16_zfill(&tile[mtile_at<T>(pos, tt)], tt < lines_ok ? base + tt * a.in_si + pos * a.in_sp : a.in,
                         tt < lines_ok);
      }
    }
    cp_async_commit();
  };
  int64_t tix = blockIdx.x;
  unsigned buf = 0, phs = 0;  // phs: parity bit of each buffer's mbarrier (TMA)
  prefetch(tix, sm);
  for (; tix < ntiles; tix += gridDim.x, buf ^= 1) {
    double2* const tile = sm + buf * X3TSmem::TILE;
    const int i0 = int(unsigned(tix) % unsigned(ntiles_i)) * T;
    const int k = int(unsigned(tix) / unsigned(ntiles_i));
    const int lines_ok = min(T, a.n_inner - i0);
    if constexpr (TMA) {
      mbar_wait(bars + buf, (phs >> buf) & 1u);
      phs ^= 1u << buf;
    } else {
      cp_async_wait0();
    }
    __syncthreads();  // this tile's copies (issued by all threads) have landed; the previous
                      // tile's t_r rows (other buffer) are read out
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int p = R * (W.k1 + 16 * (i + 8 * int(W.b))) + r;
      v[i] = (FULL || p < a.in_nvalid) ? tile[mtile_at<T>(p, t)] : make_double2(0.0, 0.0);
      v[i + 8] = (FULL || p + H < a.in_nvalid) ? tile[mtile_at<T>(p + H, t)] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // tile read by every warp: it becomes the exchange area
    prefetch(tix + gridDim.x, sm + (buf ^ 1) * X3TSmem::TILE);
    double2* const xr = tile + X3TSmem::XS * w;
    W.inverse(v, xr, lane);
    __syncwarp();
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) xr[32 * n1 + lane] = v[n1];
    nbar_sync(1 + t, 32 * R);  // line t's R t_r rows are in the area
    if (t < lines_ok) {
      const int line = i0 + t;
      double2* orow = a.out + int64_t(line) * a.out_si + int64_t(k) * a.out_sk;
      if (a.pm.n) {  // fused transpose: the row goes straight to the rank owning line (z)
        const int q = a.pm.owner(line);
        orow = a.pm.base[q] + (a.pm.off[q] + int64_t(line) * a.out_si + int64_t(k) * a.pm.sk[q]);
      }
      constexpr int XS = X3TSmem::XS;
      const double2* x = tile + XS * R * t;
      if (R == 3 && a.scale == 1.0) {
        for (int n = threadIdx.x - 32 * R * t; n < 512; n += 32 * R)
          x3_recombine<false>(x, x + XS, x + 2 * XS, n, FULL ? H : a.out_nvalid, 1.0, orow);
      } else
      for (int n = threadIdx.x - 32 * R * t; n < 512; n += 32 * R) {
        if constexpr (R == 3) {
          x3_recombine(x, x + XS, x + 2 * XS, n, FULL ? H : a.out_nvalid, a.scale, orow);
        } else if (FULL || n < a.out_nvalid) {  // x[n] = t0 + t1, n < 512
          const double2 o = cadd(x[n], x[XS + n]);
          orow[n] = a.scale == 1.0 ? o : cscale(o, a.scale);
        }
      }
    }
  }
  if constexpr (!TMA) cp_async_wait0();
  if (a.pm.n) __threadfence_system();  // remote stores performed before the following barrier
}

bool make_tile_map(CUtensorMap* map, const void* base, int64_t n_lines, int64_t n_pos, int64_t n_outer, int64_t sp,
                   int64_t sk, int T) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static const Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return Encode(nullptr);
    }
    return reinterpret_cast<Encode>(fn);
  }();
  if (!encode || T != 4 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  const cuuint64_t dims[3] = {cuuint64_t(2 * n_lines), cuuint64_t(n_pos), cuuint64_t(n_outer)};
  const cuuint64_t strides[2] = {cuuint64_t(sp) * 16, cuuint64_t(sk) * 16};
  const cuuint32_t box[3] = {cuuint32_t(2 * T), 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// c_w48 on the current device (once per device; the values do not depend on the grid)
static bool load_w48() {
  static std::atomic<uint64_t> mask{0};
  return once_per_device(mask, [] {
    double2 h[48];
    for (int e = 0; e < 48; ++e) {  // the twiddle table's expression (upload_twiddles, L = 1536, m = 32 e)
      const long double a = -2.0L * 3.141592653589793238462643383279502884L * (32 * e) / 1536;
      h[e] = make_double2(double(cosl(a)), double(sinl(a)));
    }
    return cudaMemcpyToSymbol(c_w48, h, sizeof(h)) == cudaSuccess;
  });
}

// pass C at L = 1536 (conv_r16x3): 1 launched, 0 not applicable, -1 error
int launch_conv_r16x3(fusg_ctx* ctx, const WArgs& a, cudaStream_t s) {
  static const bool on = [] {  // FUSG_CONV_R16X3=0 keeps the 64-lane radix (8, 8, 3, 8) pass C
    const char* e = getenv("FUSG_CONV_R16X3");
    return !(e && atoi(e) == 0);
  }();
  if (!on || a.in_nvalid < 1 || a.in_nvalid > 768 || a.out_nvalid > 768) return 0;
  const int64_t nl = int64_t(a.n_inner) * a.n_outer;
  if (nl >= (int64_t(1) << 31)) return 0;
  if (!load_w48()) {
    set_error(FUSG_CUDA, "pass C (1536 = 3 x 512): cannot load the W48 table");
    return -1;
  }
  // Unsharded applies, opt-in (FUSG_X3_QUADTM=1): the quad-CTA kernel with the recombination
  // through tensor memory.  Bitwise the three-warp kernel's result; measured 30.5 ms against
  // 29.4 ms at cfg5, so the three-warp kernel stays the default.
  static const bool quadtm = [] {
    const char* e = getenv("FUSG_X3_QUADTM");
    return e && atoi(e) != 0;
  }();
  if (quadtm && a.n_outer == a.ko.Px && a.n_inner == a.ko.Py && a.ko.kx_off == 0 && a.ko.kx_base == 0 &&
      a.in_sp == 1 && a.out_sp == 1 && a.ko.s_kz == 1) {
    static std::atomic<uint64_t> qattr{0};
    if (!once_per_device(qattr, [&] {
          return cudaFuncSetAttribute(conv_r16x3q, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(X3QSmem::BYTES)) == cudaSuccess;
        })) {
      set_error(FUSG_CUDA, "pass C (1536, quad CTA): cannot configure shared memory");
      return -1;
    }
    const int64_t rows = int64_t(a.ko.Py / 2 + 1) * (a.ko.Px / 2 + 1);
    const int64_t grid = std::min<int64_t>(rows, ctx->num_sms);
    conv_r16x3q<<<unsigned(grid), 384, X3QSmem::BYTES, s>>>(a);
    ctx->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
      cuda_error(err, "pass C (1536, quad CTA)");
      return -1;
    }
    return 1;
  }
  // FUSG_X3_MODE: 1 (default) input and K^ rows in two staging buffers (4 CTAs per SM); 2 one
  // shared staging buffer and lane twiddles from the tables (5 CTAs); 0 input rows from L2
  static const int mode = [] {
    const char* e = getenv("FUSG_X3_MODE");
    const int m = e ? atoi(e) : 1;
    return (m == 0 || m == 2) ? m : 1;
  }();
  const bool full = mode == 1 && a.in_nvalid == 768 && a.out_nvalid == 768;
  const auto fn = full ? conv_r16x3<1, true> : mode == 1 ? conv_r16x3<1> : mode == 2 ? conv_r16x3<2> : conv_r16x3<0>;
  const size_t smem = mode == 1 ? X3Smem<1>::BYTES : mode == 2 ? X3Smem<2>::BYTES : X3Smem<0>::BYTES;
  static std::atomic<uint64_t> attr_mask{0};
  if (!once_per_device(attr_mask, [&] {
        return cudaFuncSetAttribute(conv_r16x3<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3Smem<1>::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(conv_r16x3<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3Smem<1>::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(conv_r16x3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3Smem<2>::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(conv_r16x3<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3Smem<0>::BYTES)) == cudaSuccess;
      })) {
    set_error(FUSG_CUDA, "pass C (1536 = 3 x 512): cannot configure shared memory");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 96, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  // CTAs per resident slot (1 = fully persistent).  cfg5, one box: 1 / 2 / 4 / 8 / 16 / 32 / 64 / 128
  // -> 27.4 / 27.0 / 26.4 / 26.2 / 25.9 / 25.8 / 25.7 / 26.0 ms
  static const int waves = [] {
    const char* e = getenv("FUSG_X3_WAVES");
    return e ? std::max(1, atoi(e)) : 64;
  }();
  const int64_t grid = std::min<int64_t>(nl, int64_t(per_sm) * ctx->num_sms * waves);
  // FUSG_X3_QUAD (default 1): the (up to) four lines sharing a folded K^ row run consecutively,
  // so each row is read from DRAM about once (cfg5 pass C reads 48.4 -> 40.1 GB, apply -1 %)
  static const bool quad = [] {
    const char* e = getenv("FUSG_X3_QUAD");
    return !(e && atoi(e) == 0);
  }();
  WArgs b = a;
  if (quad) b.ko.quad = 1;
  fn<<<unsigned(grid), 96, smem, s>>>(b);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "pass C (1536 = 3 x 512)");
    return -1;
  }
  return 1;
}

// passes A/B (r2c) or D/E at L = 1536: 1 launched, 0 not applicable, -1 error
int launch_transpose_r16x3(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s) {
  // FUSG_X3_T bitmask: 1 passes A/B, 2 passes D/E (default both).  At cfg5: A 6.3 / B 10.5 /
  // D 10.9 / E 6.35 ms against 6.75 / 13.6 / 11.6 / 6.37 for the 64-lane radix (8, 8, 3, 8)
  // kernels.
  static const int mask = [] {
    const char* e = getenv("FUSG_X3_T");
    return e ? atoi(e) : 3;
  }();
  if (!(mask & (r2c ? 1 : 2))) return 0;
  if (r2c ? (a.in_nvalid > 768 || a.in_nvalid < 1 || a.in_sp != 1 || a.out_nvalid > 1536)
          : (a.out_nvalid > 768 || a.out_sp != 1 || a.in_nvalid > 1536))
    return 0;
  // FUSG_X3_TL: lines per tile.  4 (default): one CTA of 12 warps per SM, 64-byte tile segments;
  // 2: two CTAs of 6 warps per SM with 32-byte segments, measured 2x slower (A 13.4, B 25.7 ms).
  static const int T = [] {
    const char* e = getenv("FUSG_X3_TL");
    return (e && atoi(e) == 2) ? 2 : 4;
  }();
  const int64_t tiles = int64_t((a.n_inner + T - 1) / T) * a.n_outer;
  if (tiles >= (int64_t(1) << 31)) return 0;
  if (!load_w48()) {
    set_error(FUSG_CUDA, "transposing pass (1536 = 3 x 512): cannot load the W48 table");
    return -1;
  }
  // FUSG_X3_TMA=0: the column tiles move by per-thread stores / cp.async instead of tensor-map
  // box copies (T = 4, unit line stride, no peer stores, unscaled forward output)
  static const bool tma_on = [] {
    const char* e = getenv("FUSG_X3_TMA");
    return !(e && atoi(e) == 0);
  }();
  CUtensorMap tm{};
  const bool tma = tma_on && T == 4 && a.pm.n == 0 &&
                   (r2c ? (a.out_si == 1 && a.scale == 1.0 &&
                           make_tile_map(&tm, a.out, a.n_inner, a.out_nvalid, a.n_outer, a.out_sp, a.out_sk, T))
                        : (a.in_si == 1 &&
                           make_tile_map(&tm, a.in, a.n_inner, a.in_nvalid, a.n_outer, a.in_sp, a.in_sk, T)));
  using Fn = void (*)(WArgs, CUtensorMap);
  // full rows (768 valid positions on the pruned side, the whole spectrum on the other: cfg5)
#ifndef FUSG_X3T_FULL
#define FUSG_X3T_FULL 1
#endif
  const bool full = FUSG_X3T_FULL && tma && (r2c ? a.in_nvalid == 768 : (a.in_nvalid == 1536 && a.out_nvalid == 768));
  const Fn fn = T == 4 ? (r2c ? (full ? r16x3_row_to_col<4, true, 3, true> : tma ? r16x3_row_to_col<4, true> : r16x3_row_to_col<4, false>)
                              : (full ? r16x3_col_to_row<4, true, 3, true> : tma ? r16x3_col_to_row<4, true> : r16x3_col_to_row<4, false>))
                       : (r2c ? r16x3_row_to_col<2, false> : r16x3_col_to_row<2, false>);
  const size_t smem = T == 4 ? (r2c ? (tma ? X3TSmemA<4>::BYTES2 : X3TSmemA<4>::BYTES) : X3TSmemD<4>::C_BYTES)
                             : (r2c ? X3TSmemA<2>::BYTES : X3TSmemD<2>::C_BYTES);
  static std::atomic<uint64_t> attr_mask{0};
  if (!once_per_device(attr_mask, [&] {
        return cudaFuncSetAttribute(r16x3_row_to_col<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemA<4>::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_row_to_col<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemA<4>::BYTES2)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_row_to_col<4, true, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemA<4>::BYTES2)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<4, true, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemD<4>::C_BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemD<4>::C_BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemD<4>::C_BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_row_to_col<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemA<2>::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X3TSmemD<2>::C_BYTES)) == cudaSuccess;
      })) {
    set_error(FUSG_CUDA, "transposing pass (1536 = 3 x 512): cannot configure shared memory");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 96 * T, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  static const int waves = [] {  // FUSG_X3T_WAVES: CTAs per resident slot
    const char* e = getenv("FUSG_X3T_WAVES");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  const int64_t grid = std::min<int64_t>(tiles, int64_t(per_sm) * ctx->num_sms * waves);
  fn<<<unsigned(grid), 96 * T, smem, s>>>(a, tm);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "transposing pass (1536 = 3 x 512)");
    return -1;
  }
  return 1;
}

// passes A/B (r2c) or D/E at L = 1024 = 2 x 512 (the 1536 kernels with R = 2: one CTA of 8 warps
// on 4-line tiles, tensor-map TMA tiles): 1 launched, 0 not applicable, -1 error
int launch_transpose_r16x2(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s) {
  static const int mask = [] {  // FUSG_X2_T bitmask: 1 passes A/B, 2 passes D/E (default both)
    const char* e = getenv("FUSG_X2_T");
    return e ? atoi(e) : 3;
  }();
  if (!(mask & (r2c ? 1 : 2))) return 0;
  if (r2c ? (a.in_nvalid > 512 || a.in_nvalid < 1 || a.in_sp != 1 || a.out_nvalid > 1024)
          : (a.out_nvalid > 512 || a.out_sp != 1 || a.in_nvalid > 1024))
    return 0;
  constexpr int T = 4;
  const int64_t tiles = int64_t((a.n_inner + T - 1) / T) * a.n_outer;
  if (tiles >= (int64_t(1) << 31)) return 0;
  using SM2A = X3TSmemA<T, 2>;
  using SM2D = X3TSmemD<T, 2>;
  static std::atomic<uint64_t> attr_mask{0};
  if (!once_per_device(attr_mask, [] {
        double2 h[32];
        for (int e = 0; e < 32; ++e) {  // the twiddle table's expression (L = 1024, m = 32 e)
          const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (32 * e) / 1024;
          h[e] = make_double2(double(cosl(ang)), double(sinl(ang)));
        }
        return cudaMemcpyToSymbol(c_w32t, h, sizeof(h)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_row_to_col<T, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(SM2A::BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_row_to_col<T, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(SM2A::BYTES2)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<T, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(SM2D::C_BYTES)) == cudaSuccess &&
               cudaFuncSetAttribute(r16x3_col_to_row<T, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(SM2D::C_BYTES)) == cudaSuccess;
      })) {
    set_error(FUSG_CUDA, "transposing pass (1024 = 2 x 512): cannot configure the kernels");
    return -1;
  }
  static const bool tma_on = [] {
    const char* e = getenv("FUSG_X3_TMA");
    return !(e && atoi(e) == 0);
  }();
  CUtensorMap tm{};
  const bool tma = tma_on && a.pm.n == 0 &&
                   (r2c ? (a.out_si == 1 && a.scale == 1.0 &&
                           make_tile_map(&tm, a.out, a.n_inner, a.out_nvalid, a.n_outer, a.out_sp, a.out_sk, T))
                        : (a.in_si == 1 &&
                           make_tile_map(&tm, a.in, a.n_inner, a.in_nvalid, a.n_outer, a.in_sp, a.in_sk, T)));
  using Fn = void (*)(WArgs, CUtensorMap);
  const Fn fn = r2c ? (tma ? r16x3_row_to_col<T, true, 2> : r16x3_row_to_col<T, false, 2>)
                    : (tma ? r16x3_col_to_row<T, true, 2> : r16x3_col_to_row<T, false, 2>);
  const size_t smem = r2c ? (tma ? SM2A::BYTES2 : SM2A::BYTES) : SM2D::C_BYTES;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 64 * T, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  static const int waves = [] {
    const char* e = getenv("FUSG_X3T_WAVES");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  const int64_t grid = std::min<int64_t>(tiles, int64_t(per_sm) * ctx->num_sms * waves);
  fn<<<unsigned(grid), 64 * T, smem, s>>>(a, tm);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "transposing pass (1024 = 2 x 512)");
    return -1;
  }
  return 1;
}

}  // namespace fusg
