// Which formulation of one far-field pair (d2 -> rsqrt -> q*rsqrt accumulate)
// sustains the highest FP64-pipe rate on sm_100a?  Synthetic, no memory.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq64h(double x) {
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y;
}
template <int F, int NP>
__global__ void probe(double* out, int iters, const double* __restrict__ in) {
  double dz2[NP], acc[2] = {0, 0};
  double dxy2[2] = {in[threadIdx.x & 63], in[(threadIdx.x + 5) & 63]};
#pragma unroll
  for (int k = 0; k < NP; ++k) dz2[k] = in[64 + ((threadIdx.x + k) & 63)];
  const double c375 = in[128];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double q = in[(i + k) & 127];   // stand-in for the moment (LDS-like)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double d2 = dxy2[t] + dz2[k];
        const double y0 = rsq64h(d2);
        if (F == 1) {          // current: 7 FP64, two 3-register DFMAs
          const double e = fma(-(d2 * y0), y0, 1.0);
          const double c = fma(c375, e, 0.5);
          const double y = fma(y0 * e, c, y0);
          acc[t] = fma(q, y, acc[t]);
        } else if (F == 2) {   // y = y0 * (1 + e c): 8 FP64, one 3-register DFMA
          const double e = fma(-(d2 * y0), y0, 1.0);
          const double c = fma(c375, e, 0.5);
          const double y = y0 * fma(e, c, 1.0);
          acc[t] = fma(q, y, acc[t]);
        } else if (F == 3) {   // quadratic Newton (reduced precision): 6 FP64
          const double e = fma(-(d2 * y0), y0, 1.0);
          const double y = fma(y0 * e, 0.5, y0);
          acc[t] = fma(q, y, acc[t]);
        } else if (F == 4) {   // y0^2 exact first
          const double h = y0 * y0;
          const double e = fma(-d2, h, 1.0);
          const double c = fma(c375, e, 0.5);
          const double y = fma(y0 * e, c, y0);
          acc[t] = fma(q, y, acc[t]);
        } else if (F == 5) {   // split accumulators: S0 += q y0, S1 += (q y0 e) c
          const double e = fma(-(d2 * y0), y0, 1.0);
          const double c = fma(c375, e, 0.5);
          const double qy = q * y0;
          acc[t] = fma(qy * e, c, acc[t] + qy);
        }
      }
    }
    dxy2[0] += 1e-12;
    dxy2[1] += 1e-12;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1];
}
template <int F, int NP> void run(const char* name, double* d, double* in, int sms, int occ) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * occ, block = 256, iters = 400;
  probe<F, NP><<<grid, block>>>(d, 4, in);
  cudaEventRecord(e0);
  probe<F, NP><<<grid, block>>>(d, iters, in);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pairs = (double)grid * block * iters * NP * 2;
  double rate = pairs / (ms * 1e-3) / sms / 1.965e9;
  printf("{\"form\":\"%s\",\"np\":%d,\"occ\":%d,\"pairs_per_sm_clk\":%.3f,\"frac_of_7slot_roofline\":%.3f}\n",
         name, NP, occ, rate, rate * 7 / 64.0);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *d, *in; cudaMalloc(&d, sizeof(double) * sms * 8 * 256); cudaMalloc(&in, sizeof(double) * 256);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = 0.5 + 1e-3 * i; h[128] = 0.375;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int occ : {2, 4}) {
    run<1, 9>("F1_current", d, in, sms, occ);
    run<2, 9>("F2_mulp", d, in, sms, occ);
    run<3, 9>("F3_newton_quadratic", d, in, sms, occ);
    run<4, 9>("F4_h_first", d, in, sms, occ);
    run<5, 9>("F5_split_acc", d, in, sms, occ);
    run<1, 4>("F1_current", d, in, sms, occ);
  }
  return 0;
}
