// Does MUFU.RSQ64H take FP64-pipe issue slots on sm_100a?  DFMA throughput
// with one rsqrt.approx.f64 per R DFMAs (R = 8, 4, 2) against pure DFMA.
// If the MUFU were free, DFMA/SM/clk stays ~63.5; if it occupies an FP64
// slot, it drops to 63.5 R / (R + 1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix tools/fp64_mufu_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int R>
__global__ void loop(double* out, long long* clk, int iters) {
  double r[8];
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k + 1.0;
  long long c0 = clock64(); unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        r[k] = fma(r[k], r[k], 1e-9);
        if (R > 0 && (k % R) == R - 1) {
          double y;
          asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r[(k + 3) & 7]));
          acc ^= __double2hiint(y);
        }
      }
    }
  }
  long long c1 = clock64(); unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  double s = acc;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = (long long)(t1 - t0); }
}
template <int R>
void run(double* d, long long* clk, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 4, block = 256, iters = 4000;
  loop<R><<<grid, block>>>(d, clk, 100);
  cudaEventRecord(e0);
  loop<R><<<grid, block>>>(d, clk, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double n = (double)grid * block * iters * 16 * 8;
  double mhz = 1e3 * (double)h[0] / (double)h[1];
  printf("{\"dfma_per_mufu\":%d,\"ms\":%.3f,\"sm_mhz\":%.0f,\"dfma_per_sm_per_clk\":%.2f}\n", R, ms,
         mhz, n / (ms * 1e-3) / sms / (mhz * 1e6));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* d; cudaMalloc(&d, sizeof(double) * sms * 4 * 256);
  long long* clk; cudaMalloc(&clk, 16);
  run<0>(d, clk, sms);
  run<8>(d, clk, sms);
  run<4>(d, clk, sms);
  run<2>(d, clk, sms);
  run<1>(d, clk, sms);
  return 0;
}
