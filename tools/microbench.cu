// Microbenchmarks for the B200 roofline denominators this solver needs and MEASURED_PEAKS.json
// lacks: FP64 FMA/ADD throughput (Rayleigh sum, FFT butterflies), shared-memory 16-byte
// load/store throughput and warp-shuffle throughput (FFT data exchange).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dadd_kernel(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// 16-byte shared-memory stores + loads, conflict-free (consecutive lanes -> consecutive 16 B)
__global__ void smem_kernel(double* out) {
  __shared__ double2 buf[1024];
  double2 acc = make_double2(0, 0);
  const int t = threadIdx.x;
  buf[t] = make_double2(t, t);
  __syncthreads();
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    const double2 v = buf[(t + i * 32) & 1023];
    acc.x += v.x;
    buf[(t + i * 64) & 1023] = acc;  // store + load per iteration
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

// warp shuffles of 32-bit values (a double2 needs 4 of them)
__global__ void shfl_kernel(double* out) {
  int a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    a0 = __shfl_xor_sync(0xffffffffu, a0, 1) + i;
    a1 = __shfl_xor_sync(0xffffffffu, a1, 2) + i;
    a2 = __shfl_xor_sync(0xffffffffu, a2, 4) + i;
    a3 = __shfl_xor_sync(0xffffffffu, a3, 8) + i;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int blocks = sms * 8, threads = 256;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * blocks * threads));
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
  const double nthr = double(blocks) * threads;
  float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); });
  const double fma_tflops = nthr * kIters * 8 * 2 / (ms * 1e-3) / 1e12;
  ms = time_it([&] { dadd_kernel<<<blocks, threads>>>(out, 1e-3); });
  const double dadd_tops = nthr * kIters * 8 / (ms * 1e-3) / 1e12;
  ms = time_it([&] { smem_kernel<<<blocks, threads>>>(out); });
  const double smem_tbs = nthr * kIters * 32 / (ms * 1e-3) / 1e12;  // 16 B load + 16 B store
  ms = time_it([&] { shfl_kernel<<<blocks, threads>>>(out); });
  const double shfl_tbs = nthr * kIters * 4 * 4 / (ms * 1e-3) / 1e12;  // 4 x 4-byte shuffles
  CK(cudaGetLastError());
  printf("{\"sms\": %d, \"sm_clock_mhz_attr\": %d, \"fp64_fma_tflops\": %.2f, \"fp64_add_tops\": %.2f, "
         "\"smem_ldst128_tbps\": %.2f, \"shfl32_tbps\": %.2f}\n",
         sms, clk / 1000, fma_tflops, dadd_tops, smem_tbs, shfl_tbs);
  return 0;
}
