// Consumer-chain probe for the bitwise upward pass (moments.cu k_moments_bw /
// k_moments_bwc consumers): one CTA per SM, thread (k2, k3) keeps one chain
// acc += (a[k1] t2[k2]) t3[k3] over N sources whose factor records sit in
// shared memory (no producers, no barriers).  Prints cycles per source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/chain_probe.cu -o tools/chain_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int M, int UNROLL>
__global__ void probe(int n_src, int k1sel, double* out, long long* cyc) {
  constexpr int MP = (M + 1) & ~1;
  constexpr int CH = 32;
  __shared__ double sa[CH * MP], s2[CH * MP], s3[CH * MP];
  for (int i = threadIdx.x; i < CH * MP; i += blockDim.x) {
    sa[i] = 1.0 + 1e-3 * i;
    s2[i] = 1.0 - 1e-4 * i;
    s3[i] = 0.5 + 1e-5 * i;
  }
  __syncthreads();
  const int p = threadIdx.x;
  double acc = 0.0;
  const long long t0 = clock64();
  if (p < M * M) {
    const int k2 = p / M, k3 = p % M;
    for (int c = 0; c < n_src / CH; ++c) {
#pragma unroll UNROLL
      for (int jj = 0; jj < CH; ++jj) {
        const double b = __dmul_rn(sa[jj * MP + k1sel], s2[jj * MP + k2]);
        acc = __dadd_rn(acc, __dmul_rn(b, s3[jj * MP + k3]));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int n = 1 << 16;
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&cyc, 1 << 16);
  long long h[8];
  auto run = [&](auto kern, const char* name, int threads, int blocks) {
    kern<<<blocks, threads>>>(n, 3, out, cyc);
    kern<<<blocks, threads>>>(n, 3, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-32s threads %d blocks %d: %.2f cycles/source\n", name, threads, blocks,
           (double)h[0] / n);
  };
  run(probe<9, 1>, "M=9 unroll 1", 128, 148);
  run(probe<9, 4>, "M=9 unroll 4", 128, 148);
  run(probe<9, 8>, "M=9 unroll 8", 128, 148);
  run(probe<9, 32>, "M=9 unroll 32", 128, 148);
  run(probe<9, 4>, "M=9 unroll 4, 3 CTAs/SM", 128, 444);
  run(probe<9, 32>, "M=9 unroll 32, 3 CTAs/SM", 128, 444);
  run(probe<11, 4>, "M=11 unroll 4", 128, 148);
  run(probe<11, 32>, "M=11 unroll 32", 128, 148);
  return 0;
}
