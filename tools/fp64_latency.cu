// Dependent-chain latencies on one warp (clock64): DFMA, DADD, DMUL, MUFU.RSQ64H.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void lat(double* out, long long* cyc, int iters, double a) {
  double x = 1.0 + threadIdx.x * 1e-9;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      if (MODE == 0) x = fma(x, a, 1e-9);
      if (MODE == 1) x = x + a;
      if (MODE == 2) x = x * a;
      if (MODE == 3) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
    }
  }
  long long c1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
template <int MODE> void run(const char* nm, double* d, long long* c) {
  lat<MODE><<<1, 32>>>(d, c, 10, 1.0000001);
  lat<MODE><<<1, 32>>>(d, c, 1000, 1.0000001);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"op\":\"%s\",\"cycles_per_op\":%.2f}\n", nm, (double)h / (1000.0 * 32));
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1024); cudaMalloc(&c, 8);
  run<0>("dfma", d, c); run<1>("dadd", d, c); run<2>("dmul", d, c); run<3>("mufu_rsq64h+dadd", d, c);
  return 0;
}
