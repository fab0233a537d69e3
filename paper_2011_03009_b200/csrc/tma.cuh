// Tensor-map TMA for the column tiles of the transposing passes: a tile of T adjacent lines x
// P positions is a [pos][T] block of 16-byte elements whose 64-byte rows (T = 4) are swizzled
// exactly as mtile_at<4> lays them out (16-byte chunk t of row pos at t ^ ((pos >> 1) & 3)),
// which is the hardware's 64-byte swizzle mode.  One thread moves a whole tile with
// ceil(P / 256) box copies of {T lines, 256 positions}; out-of-range lines and positions are
// clipped on stores and zero-filled on loads.
#pragma once
#include <cuda.h>

#include <cstdint>

namespace fusg {

// 3-D float64 view of a field whose tile lines are adjacent complex128 elements: dim 0 =
// 2 * n_lines doubles (the line index, contiguous), dim 1 = positions (stride sp complex128
// elements), dim 2 = the outer index (stride sk).  Box {2T, 256, 1}, 64-byte swizzle (T = 4).
// Returns false when the driver entry point or the encoding is unavailable (callers fall back).
bool make_tile_map(CUtensorMap* map, const void* base, int64_t n_lines, int64_t n_pos, int64_t n_outer,
                   int64_t sp, int64_t sk, int T);

__device__ __forceinline__ void tma_store_tile_box(const CUtensorMap* map, const void* smem, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(map),
               "r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_load_tile_box(const CUtensorMap* map, void* smem, uint64_t* bar, int c0, int c1,
                                                  int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(smem))),
      "l"(map), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// the committed bulk stores have finished reading shared memory (the buffer may be rewritten)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// ... and are complete
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// generic-proxy shared-memory writes (the tile) made visible to the async proxy (the TMA store)
__device__ __forceinline__ void smem_to_async_fence() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tensor_map_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}

}  // namespace fusg
