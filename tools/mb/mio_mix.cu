// Does a warp shuffle consume the same per-SM crossbar budget as shared-memory LDS/STS?
// Kernels: (a) STS.128+LDS.128 only, (b) 4 x SHFL.32 only, (c) both interleaved.
// If (c) ~ (a) + (b) the two share one budget; if (c) ~ max(a, b) they are separate pipes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb/mio_mix tools/mb/mio_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIters = 4096;
template <bool SMEM, bool SHFL>
__global__ void mix(double* out) {
  __shared__ double2 buf[2048];
  double2 acc = make_double2(threadIdx.x, 1);
  int a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
  const int t = threadIdx.x;
  buf[t] = acc;
  buf[t + 1024] = acc;
  __syncthreads();
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    if (SMEM) {
      const double2 v = buf[(t + i * 32) & 2047];
      acc.x += v.x;
      buf[(t + i * 64) & 2047] = acc;
    }
    if (SHFL) {
      a0 = __shfl_xor_sync(0xffffffffu, a0, 1) + i;
      a1 = __shfl_xor_sync(0xffffffffu, a1, 2) + i;
      a2 = __shfl_xor_sync(0xffffffffu, a2, 4) + i;
      a3 = __shfl_xor_sync(0xffffffffu, a3, 8) + i;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + a0 + a1 + a2 + a3;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time_it = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  const float ta = time_it([&] { mix<true, false><<<blocks, threads>>>(out); });
  const float tb = time_it([&] { mix<false, true><<<blocks, threads>>>(out); });
  const float tc = time_it([&] { mix<true, true><<<blocks, threads>>>(out); });
  // crossbar bytes per warp-iteration: smem 32 lanes x 32 B = 1024 B; shfl 32 x 16 B = 512 B
  const double it = double(blocks) * (threads / 32) * kIters / sms;  // warp-iterations per SM
  printf("{\"smem_ms\": %.3f, \"shfl_ms\": %.3f, \"both_ms\": %.3f, \"smem_cyc_per_it_sm\": %.2f, "
         "\"shfl_cyc_per_it_sm\": %.2f, \"both_cyc_per_it_sm\": %.2f}\n",
         ta, tb, tc, ta * 1e-3 * 1.965e9 / it, tb * 1e-3 * 1.965e9 / it, tc * 1e-3 * 1.965e9 / it);
  return cudaGetLastError() != cudaSuccess;
}
