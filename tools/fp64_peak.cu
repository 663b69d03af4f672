// FP64 pipe microbenchmark: measures sustained DFMA throughput (the roofline
// denominator P for the interaction kernels; MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double r0 = threadIdx.x * 1e-3, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3,
         r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
      r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}
__global__ void rsqrt_loop(double* out, int iters, double a) {
  double x0 = 1.0 + threadIdx.x, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc0 += rsqrt(x0 + k); acc1 += rsqrt(x0 + k + 0.5);
      acc2 += rsqrt(x0 + k + 0.25); acc3 += rsqrt(x0 + k + 0.75);
    }
    x0 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* d; cudaMalloc(&d, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int occ : {2, 4, 8}) {
    int grid = sms * occ, block = 256;
    dfma_loop<<<grid, block>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dfma = (double)grid * block * iters * 16 * 8;
    printf("{\"probe\":\"dfma\",\"ctas_per_sm\":%d,\"ms\":%.3f,\"dfma_per_s\":%.4e,\"tflops\":%.3f,\"per_sm_per_clk_at_1965\":%.2f}\n",
           occ, ms, dfma / (ms * 1e-3), 2 * dfma / (ms * 1e-3) / 1e12, dfma / (ms * 1e-3) / sms / 1.965e9);
  }
  {
    int grid = sms * 4, block = 256; int it = 2000;
    rsqrt_loop<<<grid, block>>>(d, 10, 1e-3);
    cudaEventRecord(e0);
    rsqrt_loop<<<grid, block>>>(d, it, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * block * it * 32;
    printf("{\"probe\":\"rsqrt_f64\",\"ms\":%.3f,\"rsqrt_per_s\":%.4e}\n", ms, n / (ms * 1e-3));
  }
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, p.clockRate);
  return 0;
}
