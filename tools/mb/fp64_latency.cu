#include <cstdio>
#include <cuda_runtime.h>
template <int OP, int ILP>
__global__ void chain(double* out, double a, double b, long long* cyc) {
  double x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = a + threadIdx.x + i;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (OP == 0) x[i] = x[i] + b;
        else if (OP == 1) x[i] = fma(x[i], b, a);
        else x[i] = x[i] * b;
      }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP, int ILP>
void run(const char* name, int warps) {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  chain<OP, ILP><<<1, 32 * warps>>>(o, 1.0000001, 0.9999999, c);
  chain<OP, ILP><<<1, 32 * warps>>>(o, 1.0000001, 0.9999999, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = double(h) / (256.0 * 16);
  printf("%s ILP=%d warps/CTA=%d: %.2f cycles per dependent step (%.2f per instr per warp)\n", name, ILP, warps, per, per / ILP);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<0, 1>("DADD", 1); run<1, 1>("DFMA", 1); run<2, 1>("DMUL", 1);
  run<0, 2>("DADD", 1); run<0, 4>("DADD", 1); run<0, 8>("DADD", 1);
  run<1, 4>("DFMA", 1); run<1, 8>("DFMA", 1);
  run<0, 1>("DADD", 4); run<0, 2>("DADD", 4); run<0, 4>("DADD", 4);
  run<0, 1>("DADD", 8); run<0, 2>("DADD", 8); run<0, 4>("DADD", 8);
  run<0, 1>("DADD", 16); run<0, 2>("DADD", 16);
  return 0;
}
