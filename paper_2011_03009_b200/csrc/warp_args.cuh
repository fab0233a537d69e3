// Arguments and shared-memory geometry of the warp-engine passes (volume_potential.cu) and the
// 16x16x2 pass C (conv_r16.cu).
#pragma once
#include "internal.hpp"
#include "static_kernels.cuh"
#include "fft_warp.cuh"

namespace fusg {

struct WArgs {
  const double2* in;
  int64_t in_si, in_sk, in_sp;
  int in_nvalid;
  double2* out;
  int64_t out_si, out_sk, out_sp;
  int out_nvalid;
  double scale;
  int n_inner, n_outer;
  const double2* tw;
  KOct ko;     // pass C only
  PeerMap pm;  // fused peer-memory transpose stores (passes A and D of the sharded apply)
};

// mirror-interleaved order 0, 1, P-1, 2, P-2, ...: lines ky and Py-ky (kx and Px-kx) read the
// same folded K^ row and run close together, so the second read hits L2.
__device__ __forceinline__ int interleave_index(int r, int P) {
  if (r == 0) return 0;
  const int m = (r + 1) >> 1;
  return (r & 1) ? m : P - m;
}

// (ky, kx) of pass-C line `line` of n_inner (ky) x n_outer (kx) lines.  Unsharded (mirror) with
// quad order: the kx interleave index r runs 0 | (1, 2) | (3, 4) | ... (| Px - 1 when Px is
// even); inside a pair the two kx alternate at the finest level and ky runs mirror-interleaved,
// so the (up to) four lines reading one folded K^ row are consecutive.  Otherwise kx slow, ky
// mirror-interleaved fast (the partner kx row then follows Py lines later).
__device__ __forceinline__ void conv_line_coords(unsigned line, const KOct& ko, int n_inner, bool mirror, int& ky,
                                                 int& kx) {
  const unsigned ni = unsigned(n_inner);
  if (!mirror || !ko.quad) {
    const unsigned q = line / ni;
    ky = interleave_index(int(line - q * ni), ko.Py);
    kx = mirror ? interleave_index(int(q), ko.Px) : int(q);
    return;
  }
  if (line < ni) {
    ky = interleave_index(int(line), ko.Py);
    kx = 0;
    return;
  }
  unsigned l = line - ni;
  const unsigned npairs = unsigned(ko.Px - 1) / 2u;
  const unsigned g = l / (2u * ni);
  if (g < npairs) {
    const unsigned within = l - g * 2u * ni;
    ky = interleave_index(int(within >> 1), ko.Py);
    kx = interleave_index(int(2u * g + 1u + (within & 1u)), ko.Px);
    return;
  }
  l -= npairs * 2u * ni;  // Px even: the self-mirror column r = Px - 1 (kx = Px / 2)
  ky = interleave_index(int(l), ko.Py);
  kx = interleave_index(ko.Px - 1, ko.Px);
}

constexpr int kPPWarps = 4;  // warps per CTA
#ifndef FUSG_PP_MINB
#define FUSG_PP_MINB 3  // CTAs per SM the register budget targets (3: <= 168 registers)
#endif
// L > 512: 24+ values per lane and ~25 KB of shared memory per warp allow 2 CTAs per SM
template <int L>
constexpr int pp_min_blocks() { return L <= 512 ? FUSG_PP_MINB : 2; }

template <int L, bool PRUNED>
struct PPConvSmem {
  static constexpr int KROW = ((L / 2 + 1) + 1) & ~1;  // K^ row (L/2 + 1), padded to 32 B
  static constexpr int STAGE = PRUNED ? L / 2 : L;      // staged input positions
  static constexpr int PER_WARP = L + STAGE + KROW;      // double2 elements
  // + two mbarriers per warp (bulk staging: input row, K^ row)
  static constexpr size_t BYTES = size_t(kPPWarps) * PER_WARP * sizeof(double2) + kPPWarps * 2 * sizeof(uint64_t);
};

// pass C at L = 512 (16 x 16 x 2): 1 launched, 0 not applicable, -1 error (conv_r16.cu)
int launch_conv_r16(fusg_ctx* ctx, const WArgs& a, cudaStream_t s);
// pass C at L = 768 (3 x 16 x 16 on half-warps): 1 launched, 0 not applicable, -1 error (conv_r16x3h.cu)
int launch_conv_r16x3h(fusg_ctx* ctx, const WArgs& a, cudaStream_t s);
// pass C at L = 1024 (2 x 16 x 16 x 2): 1 launched, 0 not applicable, -1 error (conv_r16x2.cu)
int launch_conv_r16x2(fusg_ctx* ctx, const WArgs& a, cudaStream_t s);
// pass C at L = 1536 (3 x 16 x 16 x 2): 1 launched, 0 not applicable, -1 error (conv_r16x3.cu)
int launch_conv_r16x3(fusg_ctx* ctx, const WArgs& a, cudaStream_t s);
// passes A/B (r2c) or D/E at L = 1024 = 2 x 512 (conv_r16x3.cu, R = 2)
int launch_transpose_r16x2(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s);
// passes A/B (r2c) or D/E at L = 1536 (conv_r16x3.cu)
int launch_transpose_r16x3(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s);
// Passes A and B fused through an L2-resident ring of 8-plane z-slabs (conv_r16.cu)
struct ABFused {
  WArgs a;          // pass A: f rows -> ring (out = ring base; out_sk = Ny: z within the slab)
  WArgs b;          // pass B: ring -> B (in = ring base, out = bufB)
  int nz, slabs, ring;
  int64_t slot;     // elements per ring slot (Px * 8 * Ny)
  int* sync;        // [0] unused, [1 .. slabs] A tiles done, [1 + slabs ..] B tiles done
  int mode = 0;     // FUSG_ABF_MODE experiment bits
};
int launch_ab_fused_r16(fusg_ctx* ctx, const ABFused& f, cudaStream_t s);
// pass A (rows of f -> ring slot) or pass B (ring slot -> B, slot lines discarded) of one z-chunk
int launch_r16_chunk(fusg_ctx* ctx, bool pass_b, const WArgs& a, cudaStream_t s);

// passes A/B (r2c) or D/E at L = 512 (16 x 16 x 2): 1 launched, 0 not applicable, -1 error
int launch_transpose_r16(fusg_ctx* ctx, bool r2c, const WArgs& a, cudaStream_t s);

// swizzled [pos][T] column tile of the multi-line transposing passes (T = 2, 4, 8)
template <int T>
__device__ __forceinline__ int mtile_at(int pos, int t) { return pos * T + (t ^ ((pos / (8 / T)) & (T - 1))); }

}  // namespace fusg
