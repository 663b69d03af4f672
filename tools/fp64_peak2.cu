// FP64 pipe peak by instruction form (register operands matter on sm_100a):
//   0: DFMA r = r*a + b      (a, b kernel params)
//   1: DFMA r = r*r + 1e-9   (two registers + immediate)
//   2: DADD r = r + 1e-9
//   3: DMUL r = r * 0.999
//   4: DFMA r = x*y + r      (three distinct registers)
// Also reports the SM clock seen by the kernel (clock64 vs globaltimer).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void loop(double* out, long long* clk, int iters, double a, double b) {
  double r[8];
  double x = threadIdx.x * 1e-7 + 0.5, y = 1.0000001;
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  long long c0 = clock64(); unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0) r[k] = fma(r[k], a, b);
        if (MODE == 1) r[k] = fma(r[k], r[k], 1e-9);
        if (MODE == 2) r[k] = r[k] + 1e-9;
        if (MODE == 3) r[k] = r[k] * 0.999;
        if (MODE == 4) r[k] = fma(x, y, r[k]);
      }
      if (MODE == 4) { x += 1e-12; }
    }
  }
  long long c1 = clock64(); unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = (long long)(t1 - t0); }
}
template <int MODE>
void run(const char* name, double* d, long long* clk, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 4, block = 256, iters = 4000;
  loop<MODE><<<grid, block>>>(d, clk, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  loop<MODE><<<grid, block>>>(d, clk, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double n = (double)grid * block * iters * 16 * 8;
  double mhz = 1e3 * (double)h[0] / (double)h[1];
  printf("{\"form\":\"%s\",\"ms\":%.3f,\"ops_per_s\":%.4e,\"sm_mhz\":%.0f,\"per_sm_per_clk\":%.2f}\n", name, ms,
         n / (ms * 1e-3), mhz, n / (ms * 1e-3) / sms / (mhz * 1e6));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* d; cudaMalloc(&d, sizeof(double) * sms * 4 * 256);
  long long* clk; cudaMalloc(&clk, 16);
  run<0>("dfma_r_param_param", d, clk, sms);
  run<1>("dfma_r_r_imm", d, clk, sms);
  run<2>("dadd_r_imm", d, clk, sms);
  run<3>("dmul_r_imm", d, clk, sms);
  run<4>("dfma_3reg", d, clk, sms);
  return 0;
}
