// Pass C of the apply at padded z length 1024 = 2 x 512 (cfg3's z, 512^3 grids): one CTA of two
// warps per line, warp r owning the residue-r sub-transform on the 16 x 16 x 2 warp transform
// (r16.cuh), the counterpart of the 3 x 512 kernel at 1536 (conv_r16x3.cu).
//
// Forward (decimation in frequency by 2; x[n] = 0 for n >= 512 when Nz <= 512, the zero padding):
//   X[2k' + r] = DFT512_k'( y_r ),  y_r[m] = W1024^(m r) x[m],  m < 512.
// The per-lane part W1024^(lane r) of the input twiddle W1024^((32 n1 + lane) r) is merged into
// stage A's twiddle and the slot part W32^(n1 r) is a constant-bank value (residue 0 skips it).
// The spectrum is multiplied by the folded K^ row inside the last radix 2.  Inverse (decimation
// in time by 2, unnormalised, cropped to n < 512):
//   z_r = IDFT512( Z_r ),  t_r[n] = W1024^(-n r) z_r[n],  x[n] = t0[n] + t1[n].
// The two t_r rows meet in shared memory and the CTA writes the cropped row with coalesced
// stores.  Per line: one 8 KB bulk copy of the input row and one of the folded K^ row, each
// issued one line ahead; two shared exchanges plus shuffle half-exchanges per warp and direction.
// Six 2-warp CTAs (12 warps, 168 registers) share an SM.
#include <algorithm>
#include <cstdlib>

// the tan-form radix 2 inside the fused K^ multiply is a gain at 1536 only: here 7.35 vs 7.68 ms at cfg3 (spills)
#ifndef FUSG_R2_TAN_MULK
#define FUSG_R2_TAN_MULK 0
#endif
#include "r16.cuh"

namespace fusg {

// W32^j = W1024^(32 j) (the twiddle table's long-double values) for the slot twiddles
__constant__ double2 c_w32[32];

// FUSG_X2_PAD=1: exchange buffers as 16 rows of 33 entries (conflict-free for both patterns, every
// offset an immediate) instead of the XOR-swizzled [16][32].  A gain at 1536, 768 and 512; here
// (six 2-warp CTAs per SM at 168 registers) it spills 24 bytes and measures 7.44 vs 7.32 ms at
// cfg3, so it is off.
#ifndef FUSG_X2_PAD
#define FUSG_X2_PAD 0
#endif
__device__ __forceinline__ int x2_ex(int row, int col) { return FUSG_X2_PAD ? row * 33 + col : r16_ex(row, col); }
struct X2Smem {
  static constexpr int XS = FUSG_X2_PAD ? 16 * 33 : 512;  // exchange buffer of one warp
  static constexpr int XB = 0;          // [2][XS] exchange buffers, then the t_r rows
  static constexpr int KB = 2 * XS;     // folded K^ row (513, padded to 514)
  static constexpr int TW = KB + 514;   // [4][32] W512^(lane 2^j)
  static constexpr int US = TW + 128;   // [2][32] W1024^(lane r)
  static constexpr int SB = US + 64;    // staged input row (<= 512 positions)
  static constexpr int END = SB + 512;
  // + 2 mbarriers + 2 output-row offsets (left by the staging thread: the other threads skip the
  // line -> (ky, kx) divisions)
  static constexpr size_t BYTES = size_t(END) * sizeof(double2) + 4 * sizeof(uint64_t);
};

struct X2W {
  double2 u, w1, w2, w4, w8;  // W1024^(lane r); W512^(lane 2^j)
  int r, k1;
  bool b;
  __device__ __forceinline__ X2W(const double2* us, const double2* tws, int r_, int lane)
      : r(r_), k1(lane & 15), b(lane >= 16) {
    u = us[32 * r + lane];
    w1 = tws[lane];
    w2 = tws[32 + lane];
    w4 = tws[64 + lane];
    w8 = tws[96 + lane];
  }
  template <bool CONJ>
  __device__ __forceinline__ void slot_twiddle(double2* v) const {  // v[n1] *= W32^(n1 r)
    if (r == 1) {
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) v[n1] = CONJ ? cmulc(v[n1], c_w32[n1]) : cmul(v[n1], c_w32[n1]);
    }
  }
  // forward: x (zero beyond nv <= 512) -> X[2k' + r] times the folded K^ row, in the
  // half-exchanged layout (slot i: k' = k1 + 16 (i + 8 b), slot i + 8: k' + 256)
  __device__ __forceinline__ void forward_mulk(double2* v, double2* xr, int lane, const double2* kb, uint64_t* kbar,
                                               unsigned kph) const {
    slot_twiddle<false>(v);
    dft16<false>(v);
    r16_twiddle_u<false>(v, u, w1, w2, w4, w8);
#pragma unroll
    for (int k = 0; k < 16; ++k) xr[x2_ex(k, lane)] = v[k];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = xr[x2_ex(k1, 2 * h + int(b))];
    dft16<false>(v);
    mbar_wait(kbar, kph);  // this line's K^ row has landed
    // j = 2 k' + r < 512; slot i + 8 holds index j + 512, which folds to 512 - j
    r16_fwd_r2_mulk_all<32, 512>(v, b, kb, 2 * k1 + 256 * int(b) + r, std::make_integer_sequence<int, 8>{});
  }
  // inverse: Z_r -> t_r[n] = W1024^(-n r) z_r[n] in the natural layout (slot n1 = position 32 n1 + lane)
  __device__ __forceinline__ void inverse(double2* v, double2* xr, int lane) const {
    r16_r2_all<true>(v, b, std::make_integer_sequence<int, 8>{});
    dft16<true>(v);
#pragma unroll
    for (int h = 0; h < 16; ++h) xr[x2_ex(k1, 2 * h + int(b))] = v[h];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xr[x2_ex(k, lane)];
    r16_twiddle_u<true>(v, u, w1, w2, w4, w8);
    dft16<true>(v);
    slot_twiddle<true>(v);
  }
};

template <int NT>
__global__ void __launch_bounds__(64, 6) conv_r16x2(WArgs a) {
  constexpr int HZ = 513;
  extern __shared__ double2 sm[];
  const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const xb = sm + X2Smem::XB;
  double2* const xr = xb + X2Smem::XS * r;
  double2* const sb = sm + X2Smem::SB;
  double2* const kb = sm + X2Smem::KB;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + X2Smem::END);
  // tables: tws [4][32] W512^(lane 2^j) = W1024^(2 lane 2^j), us [2][32] W1024^(lane r)
  for (int e = threadIdx.x; e < 128; e += NT) sm[X2Smem::TW + e] = __ldg(a.tw + (((2 * (e & 31)) << (e >> 5)) % 1024));
  for (int e = threadIdx.x; e < 64; e += NT) sm[X2Smem::US + e] = __ldg(a.tw + (e & 31) * (e >> 5));
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const X2W W(sm + X2Smem::US, sm + X2Smem::TW, r, lane);
  const int64_t nlines = int64_t(a.n_inner) * a.n_outer;
  const int64_t stride = gridDim.x;
  const bool mirror = a.n_outer == a.ko.Px;
  auto coords = [&](int64_t line, int& ky, int& kx) { conv_line_coords(unsigned(line), a.ko, a.n_inner, mirror, ky, kx); };
  auto prefetch_in = [&](int64_t line, unsigned slot) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      reinterpret_cast<int64_t*>(bars + 2)[slot] = ky * a.out_si + int64_t(kx) * a.out_sk;
      bulk_stage(sb, a.in + ky * a.in_si + int64_t(kx) * a.in_sk, unsigned(a.in_nvalid) * sizeof(double2), bars);
    }
  };
  auto prefetch_k = [&](int64_t line) {
    if (line < nlines) {
      int ky, kx;
      coords(line, ky, kx);
      bulk_stage(kb, a.ko.line(ky, kx), HZ * sizeof(double2), bars + 1);
    }
  };
  const int nv = a.in_nvalid, onv = a.out_nvalid;
  int64_t line = blockIdx.x;
  if (threadIdx.x == 0) {
    prefetch_in(line, 0);
    prefetch_k(line);
  }
  unsigned ph = 0;  // both staging barriers complete once per line
  for (; line < nlines; line += stride, ph ^= 1) {
    double2 v[16];
    mbar_wait(bars, ph);
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) {
      const int m = 32 * n1 + lane;
      v[n1] = m < nv ? sb[m] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // the staged row is read by both warps: refill it
    if (threadIdx.x == 0) prefetch_in(line + stride, ph ^ 1u);
    W.forward_mulk(v, xr, lane, kb, bars + 1, ph);
    __syncthreads();  // K^ row read
    if (threadIdx.x == 0) prefetch_k(line + stride);
    W.inverse(v, xr, lane);
    __syncwarp();  // every lane has read its exchange slots
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) xr[32 * n1 + lane] = v[n1];
    __syncthreads();
    double2* out = a.out + reinterpret_cast<const int64_t*>(bars + 2)[ph];  // (barriers in between)
    for (int n = threadIdx.x; n < onv; n += NT) {
      const double2 o = cadd(xb[n], xb[X2Smem::XS + n]);
      out[n] = a.scale == 1.0 ? o : cscale(o, a.scale);
    }
    // (the next line's staging barrier orders these reads before its exchange writes)
  }
}

// pass C at L = 1024 (conv_r16x2): 1 launched, 0 not applicable, -1 error
int launch_conv_r16x2(fusg_ctx* ctx, const WArgs& a, cudaStream_t s) {
  static const bool on = [] {  // FUSG_CONV_R16X2=0 keeps the 64-lane radix (8, 4, 4, 8) pass C
    const char* e = getenv("FUSG_CONV_R16X2");
    return !(e && atoi(e) == 0);
  }();
  if (!on || a.in_nvalid < 1 || a.in_nvalid > 512 || a.out_nvalid > 512) return 0;
  const int64_t nl = int64_t(a.n_inner) * a.n_outer;
  if (nl >= (int64_t(1) << 31)) return 0;
  static std::atomic<uint64_t> attr_mask{0};
  if (!once_per_device(attr_mask, [] {
        double2 h[32];
        for (int e = 0; e < 32; ++e) {  // the twiddle table's expression (L = 1024, m = 32 e)
          const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (32 * e) / 1024;
          h[e] = make_double2(double(cosl(ang)), double(sinl(ang)));
        }
        return cudaMemcpyToSymbol(c_w32, h, sizeof(h)) == cudaSuccess &&
               cudaFuncSetAttribute(conv_r16x2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(X2Smem::BYTES)) == cudaSuccess;
      })) {
    set_error(FUSG_CUDA, "pass C (1024 = 2 x 512): cannot configure the kernel");
    return -1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_r16x2<64>, 64, X2Smem::BYTES) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  static const int waves = [] {  // CTAs per resident slot (1 = fully persistent); cfg3: 4 / 16 / 64 -> 7.31 / 7.21 / 7.31 ms
    const char* e = getenv("FUSG_X2_WAVES");
    return e ? std::max(1, atoi(e)) : 16;
  }();
  const int64_t grid = std::min<int64_t>(nl, int64_t(per_sm) * ctx->num_sms * waves);
  WArgs b = a;
  b.ko.quad = 1;  // the lines sharing a folded K^ row consecutive (as at 1536)
  conv_r16x2<64><<<unsigned(grid), 64, X2Smem::BYTES, s>>>(b);
  ctx->launches++;
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cuda_error(err, "pass C (1024 = 2 x 512)");
    return -1;
  }
  return 1;
}

}  // namespace fusg
