// Small in-register DFT butterflies (FP64 complex as double2) for the Stockham FFT passes.
//
// dft<R, INV>(a) replaces a[0..R) by X[q] = sum_r a[r] * exp(s*2*pi*i*r*q/R), s = -1 forward
// (FFTW_FORWARD, src/potential.cpp:138) and +1 inverse (FFTW_BACKWARD, :140), unnormalised.
// Radices: 2, 3, 4, 5, 7, 8, 16 — enough for every 7-smooth padded length.
#pragma once
#include <cuda_runtime.h>

namespace fusg {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// multiply by -i (forward quarter turn) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot90(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

namespace c {
constexpr double kS3 = 0.8660254037844386467637;   // sin(2pi/3)
constexpr double kC51 = 0.3090169943749474241023, kS51 = 0.9510565162951535721164;
constexpr double kC52 = -0.8090169943749474241023, kS52 = 0.5877852522924731291687;
constexpr double kC71 = 0.623489801858733530525, kS71 = 0.7818314824680298087084;
constexpr double kC72 = -0.2225209339563144042889, kS72 = 0.9749279121818236070181;
constexpr double kC73 = -0.9009688679024191262361, kS73 = 0.4338837391175581204758;
constexpr double kR2 = 0.7071067811865475244008;   // sqrt(2)/2
constexpr double kC16 = 0.9238795325112867561282, kS16 = 0.3826834323650897717285;
}  // namespace c

template <bool INV>
__device__ __forceinline__ void dft2(double2& a0, double2& a1) {
  const double2 t = a0;
  a0 = cadd(t, a1);
  a1 = csub(t, a1);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
  const double2 t2 = cadd(a1, a3), t3 = rot90<INV>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// multiply by w8^e, w8 = exp(-+2 pi i / 8), e in 0..7 (compile-time)
template <bool INV, int E>
__device__ __forceinline__ double2 w8(double2 a) {
  constexpr int e = E & 7;
  if constexpr (e == 0) return a;
  else if constexpr (e == 2) return rot90<INV>(a);
  else if constexpr (e == 4) return make_double2(-a.x, -a.y);
  else if constexpr (e == 6) return rot90<!INV>(a);
  else {
    // w8^1 = (r, -+r); w8^3 = (-r, -+r); w8^5 = (-r, +-r); w8^7 = (r, +-r)
    constexpr double cr = (e == 1 || e == 7) ? c::kR2 : -c::kR2;
    constexpr double ci0 = (e == 1 || e == 3) ? -c::kR2 : c::kR2;
    constexpr double ci = INV ? -ci0 : ci0;
    return make_double2(cr * a.x - ci * a.y, cr * a.y + ci * a.x);
  }
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* a) {
  // radix-2 first level: (a_r, a_{r+4})
#pragma unroll
  for (int r = 0; r < 4; ++r) dft2<INV>(a[r], a[r + 4]);
  a[5] = w8<INV, 1>(a[5]);
  a[6] = w8<INV, 2>(a[6]);
  a[7] = w8<INV, 3>(a[7]);
  dft4<INV>(a[0], a[1], a[2], a[3]);  // -> X[0],X[2],X[4],X[6]
  dft4<INV>(a[4], a[5], a[6], a[7]);  // -> X[1],X[3],X[5],X[7]
  const double2 x0 = a[0], x2 = a[1], x4 = a[2], x6 = a[3];
  const double2 x1 = a[4], x3 = a[5], x5 = a[6], x7 = a[7];
  a[0] = x0; a[1] = x1; a[2] = x2; a[3] = x3; a[4] = x4; a[5] = x5; a[6] = x6; a[7] = x7;
}

// Pruned radix-8: inputs a[4..7] are zero (zero-padded upper half), so the first radix-2
// level is a copy.
template <bool INV>
__device__ __forceinline__ void dft8_half_in(double2* a) {
#pragma unroll
  for (int r = 0; r < 4; ++r) a[r + 4] = a[r];
  a[5] = w8<INV, 1>(a[5]);
  a[6] = w8<INV, 2>(a[6]);
  a[7] = w8<INV, 3>(a[7]);
  dft4<INV>(a[0], a[1], a[2], a[3]);
  dft4<INV>(a[4], a[5], a[6], a[7]);
  const double2 x0 = a[0], x2 = a[1], x4 = a[2], x6 = a[3];
  const double2 x1 = a[4], x3 = a[5], x5 = a[6], x7 = a[7];
  a[0] = x0; a[1] = x1; a[2] = x2; a[3] = x3; a[4] = x4; a[5] = x5; a[6] = x6; a[7] = x7;
}

// Pruned radix-8: only X[0..3] are kept (cropped upper half); the last radix-4 level computes
// just its first two outputs.
template <bool INV>
__device__ __forceinline__ void dft8_half_out(double2* a) {
#pragma unroll
  for (int r = 0; r < 4; ++r) dft2<INV>(a[r], a[r + 4]);
  a[5] = w8<INV, 1>(a[5]);
  a[6] = w8<INV, 2>(a[6]);
  a[7] = w8<INV, 3>(a[7]);
  // dft4 outputs 0 and 1 only: X[2q] (q = 0, 1) from the even half, X[2q+1] from the odd half
  const double2 e0 = cadd(a[0], a[2]), e1 = csub(a[0], a[2]);
  const double2 e2 = cadd(a[1], a[3]), e3 = rot90<INV>(csub(a[1], a[3]));
  const double2 o0 = cadd(a[4], a[6]), o1 = csub(a[4], a[6]);
  const double2 o2 = cadd(a[5], a[7]), o3 = rot90<INV>(csub(a[5], a[7]));
  a[0] = cadd(e0, e2);
  a[2] = cadd(e1, e3);
  a[1] = cadd(o0, o2);
  a[3] = cadd(o1, o3);
}

// multiply by w16^e (compile-time e)
template <bool INV, int E>
__device__ __forceinline__ double2 w16(double2 a) {
  constexpr int e = E & 15;
  if constexpr ((e & 1) == 0) {
    return w8<INV, e / 2>(a);
  } else {
    // cos/sin of 2 pi e / 16 for odd e
    constexpr int q = e & 3;  // 1 or 3 within quadrant
    constexpr double cq = (q == 1) ? c::kC16 : c::kS16;
    constexpr double sq = (q == 1) ? c::kS16 : c::kC16;
    constexpr int quad = e >> 2;  // rotate by quad * 90 deg
    // base angle theta = 2 pi q/16 ; w = exp(-+ i theta) = (cq, -+sq)
    constexpr double si = INV ? sq : -sq;
    const double2 b = make_double2(cq * a.x - si * a.y, cq * a.y + si * a.x);
    if constexpr (quad == 0) return b;
    else if constexpr (quad == 1) return rot90<INV>(b);
    else if constexpr (quad == 2) return make_double2(-b.x, -b.y);
    else return rot90<!INV>(b);
  }
}

// (a + w16^E b, a - w16^E b) in 6 FMAs: w = wr (1 + i t) with the compile-time t = wi / wr, so
// w b = wr ((b.x - t b.y) + i (b.y + t b.x)) and the scale by wr rides on the butterfly's adds
// (a separate complex multiply plus the adds take 8).  Quarter turns cost 4 adds.
template <bool INV, int E>
__device__ __forceinline__ void pm16(double2 a, double2 b, double2& p, double2& m) {
  constexpr int e = E & 15;
  if constexpr (e == 0) {
    p = cadd(a, b);
    m = csub(a, b);
  } else if constexpr (e == 8) {
    p = csub(a, b);
    m = cadd(a, b);
  } else if constexpr (e == 4 || e == 12) {
    const double2 r = e == 4 ? rot90<INV>(b) : rot90<!INV>(b);
    p = cadd(a, r);
    m = csub(a, r);
  } else {
    constexpr double cs[16] = {1.0, c::kC16, c::kR2, c::kS16, 0.0, -c::kS16, -c::kR2, -c::kC16,
                               -1.0, -c::kC16, -c::kR2, -c::kS16, 0.0, c::kS16, c::kR2, c::kC16};
    constexpr double wr = cs[e];
    constexpr double sn = cs[(e + 12) & 15];  // sin(2 pi e / 16) = cos(2 pi (e - 4) / 16)
    constexpr double t = (INV ? sn : -sn) / wr;
    const double u = fma(-t, b.y, b.x), v = fma(t, b.x, b.y);
    p = make_double2(fma(wr, u, a.x), fma(wr, v, a.y));
    m = make_double2(fma(-wr, u, a.x), fma(-wr, v, a.y));
  }
}
// dft4 of (a0, w16^E1 a1, w16^E2 a2, w16^E3 a3) with the twiddles folded into the butterflies:
// w^E1 a1 +- w^E3 a3 = w^E1 (a1 +- w^(E3 - E1) a3).  20-24 FP64 instructions instead of 24-28.
template <bool INV, int E1, int E2, int E3>
__device__ __forceinline__ void dft4_tw16(double2& a0, double2& a1, double2& a2, double2& a3) {
  double2 t0, t1, s, d, o0, o1, o2, o3;
  pm16<INV, E2>(a0, a2, t0, t1);
  pm16<INV, E3 - E1 + 16>(a1, a3, s, d);
  pm16<INV, E1>(t0, s, o0, o2);
  pm16<INV, E1 + 4>(t1, d, o1, o3);  // rot90<INV>(w^E1 d) = w^(E1 + 4) d
  a0 = o0;
  a1 = o1;
  a2 = o2;
  a3 = o3;
}
// the outer level of the 4 x 4 radix 16: a[4 q1 + r2] holds B[r2][q1] before its twiddle
// w16^(r2 q1)
#ifndef FUSG_DFT16_TAN
#define FUSG_DFT16_TAN 1  // 0: multiply by the inner twiddles, then plain radix-4 butterflies
#endif
template <bool INV>
__device__ __forceinline__ void dft16_outer(double2* a) {
  if constexpr (!FUSG_DFT16_TAN) {
    a[5] = w16<INV, 1>(a[5]);
    a[6] = w16<INV, 2>(a[6]);
    a[7] = w16<INV, 3>(a[7]);
    a[9] = w16<INV, 2>(a[9]);
    a[10] = w16<INV, 4>(a[10]);
    a[11] = w16<INV, 6>(a[11]);
    a[13] = w16<INV, 3>(a[13]);
    a[14] = w16<INV, 6>(a[14]);
    a[15] = w16<INV, 9>(a[15]);
#pragma unroll
    for (int q1 = 0; q1 < 4; ++q1) dft4<INV>(a[4 * q1], a[4 * q1 + 1], a[4 * q1 + 2], a[4 * q1 + 3]);
    return;
  }
  dft4<INV>(a[0], a[1], a[2], a[3]);
  dft4_tw16<INV, 1, 2, 3>(a[4], a[5], a[6], a[7]);
  dft4_tw16<INV, 2, 4, 6>(a[8], a[9], a[10], a[11]);
  dft4_tw16<INV, 3, 6, 9>(a[12], a[13], a[14], a[15]);
}

template <bool INV>
__device__ __forceinline__ void dft16(double2* a) {
  // 4 x 4: inner DFT4 over stride-4 inputs, twiddle, outer DFT4
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) dft4<INV>(a[r2], a[r2 + 4], a[r2 + 8], a[r2 + 12]);
  // a[r2 + 4*q1] now holds B[r2][q1]; the twiddles w16^(r2*q1) ride on the outer butterflies
  dft16_outer<INV>(a);
  // X[q1 + 4 q2] = a[4 q1 + q2]  -> transpose 4x4
  double2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = a[i];
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) a[q1 + 4 * q2] = t[4 * q1 + q2];
}

// Pruned radix-16: inputs a[8..15] are zero (zero-padded upper half), so each inner DFT4
// sees two inputs.
template <bool INV>
__device__ __forceinline__ void dft16_half_in(double2* a) {
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) {
    const double2 x0 = a[r2], x1 = a[r2 + 4], x1r = rot90<INV>(x1);
    a[r2] = cadd(x0, x1);
    a[r2 + 4] = cadd(x0, x1r);
    a[r2 + 8] = csub(x0, x1);
    a[r2 + 12] = csub(x0, x1r);
  }
  dft16_outer<INV>(a);
  double2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = a[i];
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) a[q1 + 4 * q2] = t[4 * q1 + q2];
}

// Pruned radix-16: only X[0..7] are kept (cropped upper half) in a[0..7].
template <bool INV>
__device__ __forceinline__ void dft16_half_out(double2* a) {
#pragma unroll
  for (int r2 = 0; r2 < 4; ++r2) dft4<INV>(a[r2], a[r2 + 4], a[r2 + 8], a[r2 + 12]);
  // outer DFT4 over a[4 q1 .. 4 q1 + 3], outputs q2 = 0, 1 only: X[q1 + 4 q2] (the unused
  // differences of the fused butterflies are dead code)
  dft16_outer<INV>(a);
  double2 x[8];
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1) {
    x[q1] = a[4 * q1];
    x[q1 + 4] = a[4 * q1 + 1];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x[i];
}

// multiply by w32^e, w32 = exp(-+2 pi i / 32), e in 0..7 (compile-time)
template <bool INV, int E>
__device__ __forceinline__ double2 w32(double2 a) {
  static_assert(E >= 0 && E < 8, "w32: e in 0..7");
  if constexpr ((E & 1) == 0) {
    return w16<INV, E / 2>(a);
  } else {
    // cos, sin of 2 pi e / 32 for odd e
    constexpr double cs[4] = {0.98078528040323044912618, 0.83146961230254523707879, 0.55557023301960222474283,
                              0.19509032201612826784828};
    constexpr double cq = cs[E / 2], sq = cs[3 - E / 2];
    constexpr double si = INV ? sq : -sq;  // w = (cq, -+sq)
    return make_double2(cq * a.x - si * a.y, cq * a.y + si * a.x);
  }
}

template <bool INV>
__device__ __forceinline__ void dft3(double2* a) {
  const double2 t1 = cadd(a[1], a[2]);
  const double2 t2 = csub(a[1], a[2]);
  const double2 m1 = make_double2(a[0].x - 0.5 * t1.x, a[0].y - 0.5 * t1.y);
  const double2 m2 = rot90<INV>(cscale(t2, c::kS3));
  a[0] = cadd(a[0], t1);
  a[1] = cadd(m1, m2);
  a[2] = csub(m1, m2);
}

template <bool INV>
__device__ __forceinline__ void dft5(double2* a) {
  const double2 t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
  const double2 t3 = csub(a[1], a[4]), t4 = csub(a[2], a[3]);
  const double2 a0 = a[0];
  const double2 m1 = make_double2(a0.x + c::kC51 * t1.x + c::kC52 * t2.x, a0.y + c::kC51 * t1.y + c::kC52 * t2.y);
  const double2 m2 = make_double2(a0.x + c::kC52 * t1.x + c::kC51 * t2.x, a0.y + c::kC52 * t1.y + c::kC51 * t2.y);
  const double2 n1 = rot90<INV>(make_double2(c::kS51 * t3.x + c::kS52 * t4.x, c::kS51 * t3.y + c::kS52 * t4.y));
  const double2 n2 = rot90<INV>(make_double2(c::kS52 * t3.x - c::kS51 * t4.x, c::kS52 * t3.y - c::kS51 * t4.y));
  a[0] = make_double2(a0.x + t1.x + t2.x, a0.y + t1.y + t2.y);
  a[1] = cadd(m1, n1);
  a[4] = csub(m1, n1);
  a[2] = cadd(m2, n2);
  a[3] = csub(m2, n2);
}

template <bool INV>
__device__ __forceinline__ void dft7(double2* a) {
  const double2 p1 = cadd(a[1], a[6]), p2 = cadd(a[2], a[5]), p3 = cadd(a[3], a[4]);
  const double2 q1 = csub(a[1], a[6]), q2 = csub(a[2], a[5]), q3 = csub(a[3], a[4]);
  const double2 a0 = a[0];
  // m_q = a0 + sum_j cos(2 pi j q / 7) p_j ; n_q = -+i sum_j sin(2 pi j q/7) q_j
  const double2 m1 = make_double2(a0.x + c::kC71 * p1.x + c::kC72 * p2.x + c::kC73 * p3.x,
                                  a0.y + c::kC71 * p1.y + c::kC72 * p2.y + c::kC73 * p3.y);
  const double2 m2 = make_double2(a0.x + c::kC72 * p1.x + c::kC73 * p2.x + c::kC71 * p3.x,
                                  a0.y + c::kC72 * p1.y + c::kC73 * p2.y + c::kC71 * p3.y);
  const double2 m3 = make_double2(a0.x + c::kC73 * p1.x + c::kC71 * p2.x + c::kC72 * p3.x,
                                  a0.y + c::kC73 * p1.y + c::kC71 * p2.y + c::kC72 * p3.y);
  // sin(2pi*jq/7): q=1: s1,s2,s3 ; q=2: s2,-s3,-s1 ; q=3: s3,-s1,s2
  const double2 n1 = rot90<INV>(make_double2(c::kS71 * q1.x + c::kS72 * q2.x + c::kS73 * q3.x,
                                             c::kS71 * q1.y + c::kS72 * q2.y + c::kS73 * q3.y));
  const double2 n2 = rot90<INV>(make_double2(c::kS72 * q1.x - c::kS73 * q2.x - c::kS71 * q3.x,
                                             c::kS72 * q1.y - c::kS73 * q2.y - c::kS71 * q3.y));
  const double2 n3 = rot90<INV>(make_double2(c::kS73 * q1.x - c::kS71 * q2.x + c::kS72 * q3.x,
                                             c::kS73 * q1.y - c::kS71 * q2.y + c::kS72 * q3.y));
  a[0] = make_double2(a0.x + p1.x + p2.x + p3.x, a0.y + p1.y + p2.y + p3.y);
  a[1] = cadd(m1, n1);
  a[6] = csub(m1, n1);
  a[2] = cadd(m2, n2);
  a[5] = csub(m2, n2);
  a[3] = cadd(m3, n3);
  a[4] = csub(m3, n3);
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2* a) {
  if constexpr (R == 2) dft2<INV>(a[0], a[1]);
  else if constexpr (R == 3) dft3<INV>(a);
  else if constexpr (R == 4) dft4<INV>(a[0], a[1], a[2], a[3]);
  else if constexpr (R == 5) dft5<INV>(a);
  else if constexpr (R == 7) dft7<INV>(a);
  else if constexpr (R == 8) dft8<INV>(a);
  else if constexpr (R == 16) dft16<INV>(a);
  else static_assert(R == 2, "unsupported radix");
}

}  // namespace fusg
