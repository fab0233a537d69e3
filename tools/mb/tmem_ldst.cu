// TMEM as lane-private scratch: throughput of tcgen05.st / tcgen05.ld (32x32b.x64) per SM for 4, 8, 12
// warps per CTA (one CTA per SM, 512 columns).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st64(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
      "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};\n" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(v[32]), "r"(v[33]), "r"(v[34]), "r"(v[35]), "r"(v[36]),
      "r"(v[37]), "r"(v[38]), "r"(v[39]), "r"(v[40]), "r"(v[41]), "r"(v[42]), "r"(v[43]), "r"(v[44]), "r"(v[45]),
      "r"(v[46]), "r"(v[47]), "r"(v[48]), "r"(v[49]), "r"(v[50]), "r"(v[51]), "r"(v[52]), "r"(v[53]), "r"(v[54]),
      "r"(v[55]), "r"(v[56]), "r"(v[57]), "r"(v[58]), "r"(v[59]), "r"(v[60]), "r"(v[61]), "r"(v[62]), "r"(v[63])
      : "memory");
}
__device__ __forceinline__ void tm_ld64(uint32_t addr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32]),
        "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]), "=r"(v[40]),
        "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]),
        "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]),
        "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
      : "r"(addr)
      : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// mode 0: st + ld alternating; 1: st only; 2: ld only
__global__ void __launch_bounds__(384, 1) tmem_bench(int iters, int mode, long long* cycles, uint32_t* sink, int* ok) {
  __shared__ uint32_t base_s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = base_s;
  // warp w owns lanes 32 (w % 4) .. + 31 and columns 128 (w / 4) .. + 127 (two x64 blocks)
  const uint32_t addr = base + (uint32_t(32 * (w & 3)) << 16) + 128u * uint32_t(w >> 2);
  uint32_t v[64], u[64];
  for (int i = 0; i < 64; ++i) v[i] = threadIdx.x * 64u + i + blockIdx.x;
  // correctness: write, read back
  tm_st64(addr, v);
  tm_wait_st();
  tm_ld64(addr, u);
  tm_wait_ld();
  bool good = true;
  for (int i = 0; i < 64; ++i) good = good && (u[i] == v[i]);
  if (!good) atomicExch(ok, 0);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode != 2) {
      tm_st64(addr + 64u * (it & 1), v);
      tm_wait_st();
    }
    if (mode != 1) {
      tm_ld64(addr + 64u * (it & 1), u);
      tm_wait_ld();
      for (int i = 0; i < 64; ++i) v[i] ^= u[i];
    } else {
      for (int i = 0; i < 64; ++i) v[i] += it;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 64; ++i) s ^= v[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base));
}

int main() {
  long long* cyc;
  uint32_t* sink;
  int* ok;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 384 * sizeof(uint32_t));
  cudaMalloc(&ok, sizeof(int));
  const int one = 1;
  cudaMemcpy(ok, &one, sizeof(int), cudaMemcpyHostToDevice);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 12}) {
      tmem_bench<<<148, 32 * warps>>>(iters, mode, cyc, sink, ok);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      int hok = 0;
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      cudaMemcpy(&hok, ok, sizeof(int), cudaMemcpyDeviceToHost);
      const double bytes = double(iters) * warps * 64 * 32 * 4;  // per direction per SM
      printf("{\"mode\": \"%s\", \"warps\": %d, \"err\": \"%s\", \"roundtrip_ok\": %d, \"cycles\": %lld, \"bytes_per_clk_per_SM_per_direction\": %.1f}\n",
             mode == 0 ? "st+ld" : mode == 1 ? "st" : "ld", warps, cudaGetErrorString(e), hok, h[0], bytes / double(h[0]));
    }
  return 0;
}
