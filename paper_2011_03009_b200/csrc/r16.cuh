// 16 x 16 x 2 warp transform pieces shared by the L = 512 kernels (conv_r16.cu) and the
// L = 1536 = 3 x 512 (conv_r16x3.cu) and L = 1024 = 2 x 512 (conv_r16x2.cu) kernels.
#pragma once
#include <utility>

#include "warp_args.cuh"

namespace fusg {

// TAB = false: from four exact table powers [w1, w2, w4, w8][lane] (<= 3 products);
// TAB = true: all fifteen from an exact [k][lane] table (more shared loads, fewer FP64 ops).
// Either table lives in shared memory, shared by the CTA's warps.
template <bool CONJ>
__device__ __forceinline__ void r16_twiddle(double2* v, double2 w1, double2 w2, double2 w4, double2 w8) {
  auto m = [](double2 x, double2 t) { return CONJ ? cmulc(x, t) : cmul(x, t); };
  const double2 w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
  v[1] = m(v[1], w1);
  v[2] = m(v[2], w2);
  v[3] = m(v[3], w3);
  v[4] = m(v[4], w4);
  v[5] = m(v[5], w5);
  v[6] = m(v[6], w6);
  v[7] = m(v[7], w7);
  v[8] = m(v[8], w8);
  v[9] = m(v[9], cmul(w8, w1));
  v[10] = m(v[10], cmul(w8, w2));
  v[11] = m(v[11], cmul(w8, w3));
  v[12] = m(v[12], cmul(w8, w4));
  v[13] = m(v[13], cmul(w8, w5));
  v[14] = m(v[14], cmul(w8, w6));
  v[15] = m(v[15], cmul(w8, w7));
}

template <bool TAB>
struct R16Tw {  // W512^(n2 k) for k = 1..15
  const double2* t;
  int lane;
  template <bool CONJ>
  __device__ __forceinline__ void apply(double2* v) const {
    auto m = [](double2 x, double2 t) { return CONJ ? cmulc(x, t) : cmul(x, t); };
    if constexpr (TAB) {
#pragma unroll
      for (int k = 1; k < 16; ++k) v[k] = m(v[k], t[32 * k + lane]);
      return;
    }
    r16_twiddle<CONJ>(v, t[lane], t[32 + lane], t[64 + lane], t[96 + lane]);
  }
};

__device__ __forceinline__ double2 shfl_xor_d2(double2 x, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, x.x, m), __shfl_xor_sync(0xffffffffu, x.y, m));
}
__device__ __forceinline__ double2 sel_d2(bool p, double2 a, double2 b) { return p ? a : b; }

// v[k] *= u * W512^(lane k), k = 0..15, from u and the exact powers w1, w2, w4, w8 (CONJ: by the
// conjugates)
template <bool CONJ>
__device__ __forceinline__ void r16_twiddle_u(double2* v, double2 u, double2 w1, double2 w2, double2 w4, double2 w8) {
  auto m = [](double2 x, double2 t) { return CONJ ? cmulc(x, t) : cmul(x, t); };
  // each power p_k = u W512^(lane k) is applied to v[k] and, times w8, to v[k + 8] as soon as it
  // exists, so few products are live at once
  v[0] = m(v[0], u);
  const double2 p8 = cmul(u, w8);
  v[8] = m(v[8], p8);
  const double2 p1 = cmul(u, w1);
  v[1] = m(v[1], p1);
  v[9] = m(v[9], cmul(p1, w8));
  const double2 p2 = cmul(u, w2);
  v[2] = m(v[2], p2);
  v[10] = m(v[10], cmul(p2, w8));
  const double2 p4 = cmul(u, w4);
  v[4] = m(v[4], p4);
  v[12] = m(v[12], cmul(p4, w8));
  const double2 p3 = cmul(p1, w2);
  v[3] = m(v[3], p3);
  v[11] = m(v[11], cmul(p3, w8));
  const double2 p5 = cmul(p1, w4);
  v[5] = m(v[5], p5);
  v[13] = m(v[13], cmul(p5, w8));
  const double2 p6 = cmul(p2, w4);
  v[6] = m(v[6], p6);
  v[14] = m(v[14], cmul(p6, w8));
  const double2 p7 = cmul(p3, w4);
  v[7] = m(v[7], p7);
  v[15] = m(v[15], cmul(p7, w8));
}

#ifndef FUSG_R2_TAN_MULK
#define FUSG_R2_TAN_MULK 1  // the tan form inside pass C's fused radix 2 + K^ multiply only
#endif
#ifndef FUSG_R2_TAN
#define FUSG_R2_TAN 0  // 1: z0 +- w z1 in tan form (6 FP64 instructions per step instead of 8, but the
                       // per-lane-half (wr, t) selects cost issue slots: cfg5 passes A / B 4.19 / 8.36 -> 4.33 / 8.63 ms,
                       // pass C unchanged)
#endif
// radix 2 over n2lo with twiddle W32^(q1 n2lo), q1 = i + 8 b (forward), and its adjoint
template <int I, bool TAN = (FUSG_R2_TAN != 0)>
__device__ __forceinline__ void r16_fwd_r2(double2* v, bool b) {
  const double2 send = sel_d2(b, v[I], v[I + 8]);  // lane b keeps q1 in [8b, 8b + 8)
  const double2 recv = shfl_xor_d2(send, 16);
  const double2 z0 = sel_d2(b, recv, v[I]);
  const double2 z1 = sel_d2(b, v[I + 8], recv);
  if constexpr (I == 0 || !TAN) {
    double2 t = w32<false, I>(z1);
    t = sel_d2(b, rot90<false>(t), t);  // W32^8 = -i
    v[I] = cadd(z0, t);
    v[I + 8] = csub(z0, t);
  } else {
    // z0 +- w z1, w = W32^(I + 8 b) = wr (1 + i t): the two compile-time (wr, t) pairs are picked
    // by the lane half and the scale rides on the butterfly (6 FMAs; multiply then add: 8)
    constexpr double cs[9] = {1.0, 0.98078528040323044912618, c::kC16, 0.83146961230254523707879, c::kR2,
                              0.55557023301960222474283, c::kS16, 0.19509032201612826784828, 0.0};
    constexpr double co = cs[I], si = cs[8 - I];  // cos, sin of 2 pi I / 32; w(b = 0) = (co, -si), w(b = 1) = (-si, -co)
    const double wr = b ? -si : co;
    const double t = b ? co / si : -si / co;
    const double u = fma(-t, z1.y, z1.x), w = fma(t, z1.x, z1.y);
    v[I] = make_double2(fma(wr, u, z0.x), fma(wr, w, z0.y));
    v[I + 8] = make_double2(fma(-wr, u, z0.x), fma(-wr, w, z0.y));
  }
}
template <int I>
__device__ __forceinline__ void r16_inv_r2(double2* v, bool b) {
  const double2 z0 = cadd(v[I], v[I + 8]);
  double2 z1 = w32<true, I>(csub(v[I], v[I + 8]));
  z1 = sel_d2(b, rot90<true>(z1), z1);
  const double2 send = sel_d2(b, z0, z1);  // lane b collects Z_b[q1] for every q1
  const double2 recv = shfl_xor_d2(send, 16);
  v[I] = sel_d2(b, recv, z0);
  v[I + 8] = sel_d2(b, z1, recv);
}
// The forward cross-lane radix 2 fused with the spectral multiply by a folded K^ row in shared
// memory: after step I, slot I is multiplied by kb[p0 + STEP I] and slot I + 8 by its mirror
// kb[MIR - p0 - STEP I].  The two K^ values of step I + 1 are loaded before step I's
// half-exchange, so their shared-load latency hides behind the shuffle (a separate multiply
// loop waits on every load).
template <int STEP, int MIR, int I>
__device__ __forceinline__ void r16_fwd_r2_mulk(double2* v, bool b, const double2* kb, int p0, double2& ka,
                                                double2& kz) {
  double2 na, nz;
  if constexpr (I + 1 < 8) {
    const int p = p0 + STEP * (I + 1);
    na = kb[p];
    nz = kb[MIR - p];
  }
  r16_fwd_r2<I, (FUSG_R2_TAN_MULK != 0)>(v, b);
  v[I] = cmul(v[I], ka);
  v[I + 8] = cmul(v[I + 8], kz);
  if constexpr (I + 1 < 8) {
    ka = na;
    kz = nz;
  }
}
template <int STEP, int MIR, int... Is>
__device__ __forceinline__ void r16_fwd_r2_mulk_all(double2* v, bool b, const double2* kb, int p0,
                                                    std::integer_sequence<int, Is...>) {
  double2 ka = kb[p0], kz = kb[MIR - p0];
  (r16_fwd_r2_mulk<STEP, MIR, Is>(v, b, kb, p0, ka, kz), ...);
}

template <bool INV, int... Is>
__device__ __forceinline__ void r16_r2_all(double2* v, bool b, std::integer_sequence<int, Is...>) {
  if constexpr (INV) (r16_inv_r2<Is>(v, b), ...);
  else (r16_fwd_r2<Is>(v, b), ...);
}

__device__ __forceinline__ int r16_ex(int row, int col) { return row * 32 + (col ^ (row & 7)); }

}  // namespace fusg
