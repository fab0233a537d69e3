// Compile-time-planned Stockham stages for the hot padded lengths.
//
// Same algorithm and endpoint interface as fft_pass.cuh, but the radix sequence, stride
// products, twiddle strides and threads-per-line are template constants: index arithmetic
// folds to shifts/multiplies by constants, the guards vanish when the thread count divides
// the butterfly count, and nothing is indexed dynamically (no local-memory plan copy).
#pragma once
#include "fft_pass.cuh"

namespace fusg {

template <int... Rs>
struct Radices {
  static constexpr int n = sizeof...(Rs);
  static constexpr int r[n] = {Rs...};
  static constexpr int at(int s) { return r[s]; }
  static constexpr int ns(int s) {  // product of radices before stage s
    int p = 1;
    for (int i = 0; i < s; ++i) p *= r[i];
    return p;
  }
  static constexpr int len() { return ns(n); }
  static constexpr int tpl() {  // threads per line so that no thread holds > kMaxElems values
    int t = 1;
    for (int i = 0; i < n; ++i) {
      const int nb = len() / r[i];
      const int b = kMaxElems / r[i];
      const int need = (nb + b - 1) / b;
      t = need > t ? need : t;
    }
    return t;
  }
};

template <int L, int TPL, int T, bool INV, int R, int NS, bool FIRST, bool LAST, class Src, class Dst>
__device__ __forceinline__ void stage_s(double2* sm, int t, int jt, const double2* __restrict__ tw,
                                        Src& src, Dst& dst) {
  constexpr int NB = L / R;
  constexpr int B = kMaxElems / R;
  constexpr int TWS = L / (NS * R);
  constexpr bool EXACT = (B * TPL == NB);  // every (thread, b) slot is a real butterfly
  double2 v[kMaxElems];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = jt + b * TPL;
    const bool ok = EXACT || j < NB;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int pos = j + r * NB;
      double2 x = make_double2(0.0, 0.0);
      if (ok) x = FIRST ? src.load(pos, b * R + r) : sm[tidx<T>(pos, t)];
      v[b * R + r] = x;
    }
  }
  if constexpr ((!FIRST || Src::kSmem) && (!LAST || Dst::kSmem)) __syncthreads();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = jt + b * TPL;
    const bool ok = EXACT || j < NB;
    const int k = (NS > 1) ? j % NS : 0;
    if constexpr (NS > 1) {
      if (ok) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const double2 w = tw[r * k * TWS];  // shared or global table
          v[b * R + r] = INV ? cmulc(v[b * R + r], w) : cmul(v[b * R + r], w);
        }
      }
    }
    dft<R, INV>(v + b * R);
    if (ok) {
      const int base = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int p = base + r * NS;
        if constexpr (LAST) dst.store(p, b * R + r, v[b * R + r]);
        else sm[tidx<T>(p, t)] = v[b * R + r];
      }
    }
  }
  if constexpr (!LAST) __syncthreads();
}

template <class RL, int T, bool INV, int S = 0, class Src, class Dst>
__device__ __forceinline__ void fft_line_s(double2* sm, int t, int jt, const double2* __restrict__ tw,
                                           Src& src, Dst& dst) {
  if constexpr (S < RL::n) {
    stage_s<RL::len(), RL::tpl(), T, INV, RL::at(S), RL::ns(S), S == 0, S == RL::n - 1>(
        sm, t, jt, tw, src, dst);
    fft_line_s<RL, T, INV, S + 1>(sm, t, jt, tw, src, dst);
  }
}

template <class RL>
__device__ __forceinline__ int first_stage_pos_s(int jt, int e) {
  constexpr int R = RL::at(0);
  constexpr int NB = RL::len() / R;
  const int b = e / R, r = e - (e / R) * R;
  const int j = jt + b * RL::tpl();
  return (b < kMaxElems / R && j < NB) ? j + r * NB : -1;
}

}  // namespace fusg
