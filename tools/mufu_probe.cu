// Throughput probes for the pieces of an FP64 reciprocal square root on sm_100a:
// MUFU.RSQ64H (rsqrt.approx.f64), MUFU.RSQ (f32), F2F conversions, and full rsqrt variants.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq64h(double x) {
  double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y;
}
template <int MODE>
__global__ void probe(double* out, int iters, double step) {
  double x[8], acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = 1.0 + threadIdx.x + 0.1 * k; acc[k] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) {           // MUFU.RSQ64H only: feed result back as next input
        x[k] = rsq64h(x[k]);
      } else if (MODE == 1) {    // f32 MUFU.RSQ only
        float f = __int_as_float(__double2hiint(x[k])); f = rsqrtf(f); x[k] = __hiloint2double(__float_as_int(f), 0);
      } else if (MODE == 2) {    // F2F f64->f32->f64 round trip
        float f = __double2float_rn(x[k]); x[k] = (double)f + 1.0;
      } else if (MODE == 3) {    // full MUFU seed + 1 cubic correction (5 FP64 ops)
        double y = rsq64h(x[k]);
        double e = fma(-x[k] * y, y, 1.0);
        double c = fma(0.375, e, 0.5);
        y = fma(y * e, c, y);
        acc[k] += y; x[k] += step;
      } else if (MODE == 4) {    // libdevice exp
        acc[k] += exp(-x[k]); x[k] += step;
      } else if (MODE == 5) {    // integer-seeded rsqrt: magic seed + 3 Newton (no MUFU)
        double xx = x[k];
        int hi = 0x5fe6eb50 - (__double2hiint(xx) >> 1);
        double y = __hiloint2double(hi, 0);
        double hx = 0.5 * xx;
        y = y * fma(-hx * y, y, 1.5);
        y = y * fma(-hx * y, y, 1.5);
        double e = fma(-xx * y, y, 1.0);
        double c = fma(0.375, e, 0.5);
        y = fma(y * e, c, y);
        acc[k] += y; x[k] += step;
      } else if (MODE == 6) {    // plain DADD chain reference
        acc[k] += x[k]; x[k] += step;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k] + x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(const char* name, double* d, int sms, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 4, block = 256;
  probe<MODE><<<grid, block>>>(d, 10, 1e-6);
  cudaEventRecord(e0);
  probe<MODE><<<grid, block>>>(d, iters, 1e-6);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)grid * block * iters * 8;
  printf("{\"probe\":\"%s\",\"ms\":%.3f,\"ops_per_s\":%.4e,\"per_sm_per_clk_1965\":%.3f}\n", name, ms,
         n / (ms * 1e-3), n / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* d; cudaMalloc(&d, sizeof(double) * sms * 4 * 256);
  run<0>("mufu_rsq64h", d, sms, 4000);
  run<1>("mufu_rsq_f32", d, sms, 4000);
  run<2>("f2f_roundtrip", d, sms, 4000);
  run<3>("rsqrt_mufu_cubic", d, sms, 4000);
  run<4>("exp_f64", d, sms, 1000);
  run<5>("rsqrt_intseed", d, sms, 4000);
  run<6>("dadd_chain", d, sms, 4000);
  return 0;
}
