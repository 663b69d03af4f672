// Microbenchmarks for FP64 instruction-mix throughput on sm_100a: is a DFMA with
// three distinct register operands slower than one with an immediate / reused
// operand (register-file bank limits), and does MUFU.RSQ64H steal FP64 issue?
#include <cstdio>
#include <cuda_runtime.h>
#define N 8
__device__ __forceinline__ double rsq64h(double x) {
  double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y;
}
template <int MODE>
__global__ void probe(double* out, int iters, const double* __restrict__ ab) {
  double r[N], a[N], b[N];
#pragma unroll
  for (int k = 0; k < N; ++k) { r[k] = threadIdx.x * 1e-3 + k; a[k] = ab[(threadIdx.x + k) & 63]; b[k] = ab[64 + ((threadIdx.x * 3 + k) & 63)]; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (MODE == 0) r[k] = fma(r[k], a[k], b[k]);          // 3 distinct regs
        if (MODE == 1) r[k] = fma(r[k], a[k], 0.5);           // 2 regs + imm
        if (MODE == 2) r[k] = r[k] * a[k];                    // DMUL 2 regs
        if (MODE == 3) { double y = rsq64h(r[k]); r[k] = fma(y, a[k], b[k]); }      // MUFU + 3-reg DFMA
        if (MODE == 4) { double y = rsq64h(r[k]); r[k] = fma(y, a[k], 0.5); }       // MUFU + imm DFMA
        if (MODE == 5) { double y = r[k] * a[k]; r[k] = fma(y, b[k], 0.25); }       // no MUFU
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int k = 0; k < N; ++k) t += r[k] + a[k] + b[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE> void run(const char* name, double* d, int sms, int per, double fp64_per, double mufu_per) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 4, block = 256, iters = 2000;
  probe<MODE><<<grid, block>>>(d, 10, d + grid * block);
  cudaEventRecord(e0);
  probe<MODE><<<grid, block>>>(d, iters, d + grid * block);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)grid * block * iters * 8 * N;  // inner bodies
  double rate = n / (ms * 1e-3) / sms / 1.965e9;    // bodies per clk per SM at 1965
  printf("{\"probe\":\"%s\",\"ms\":%.3f,\"bodies_per_sm_clk\":%.3f,\"fp64_per_sm_clk\":%.2f,\"mufu_per_sm_clk\":%.2f}\n",
         name, ms, rate, rate * fp64_per, rate * mufu_per);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, sizeof(double) * (sms * 4 * 256 + 128));
  double h[128]; for (int i = 0; i < 64; ++i) { h[i] = 1.0 + 1e-9 * i; h[64 + i] = 1e-9 * (i + 1); }
  cudaMemcpy(d + sms * 4 * 256, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>("dfma_3reg", d, sms, 0, 1, 0);
    run<1>("dfma_2reg_imm", d, sms, 0, 1, 0);
    run<2>("dmul_2reg", d, sms, 0, 1, 0);
    run<3>("mufu_dfma3", d, sms, 0, 1, 1);
    run<4>("mufu_dfma_imm", d, sms, 0, 1, 1);
    run<5>("dmul_dfma_imm", d, sms, 0, 2, 0);
  }
  return 0;
}
