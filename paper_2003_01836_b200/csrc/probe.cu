// FP64-pipe roofline denominator, measured live: sustained DFMA throughput of
// the device (MEASURED_PEAKS.json carries HBM and bf16 peaks only).
#include "bltc_internal.cuh"
#include "libm_exp.cuh"

namespace bltc {
namespace {
__global__ void k_dfma_loop(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_libm_exp(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = libm_exp(x[i]);
}
}  // namespace
}  // namespace bltc

extern "C" BLTC_API int bltc_probe_fp64(int device, double seconds, double* dfma_per_s) {
  using namespace bltc;
  try {
    if (device >= 0) BLTC_CUDA(cudaSetDevice(device));
    int dev = 0, sms = 0;
    BLTC_CUDA(cudaGetDevice(&dev));
    BLTC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = sms * 4, block = 256;
    double* d = nullptr;
    BLTC_CUDA(cudaMalloc(&d, sizeof(double) * grid * block));
    cudaEvent_t e0, e1;
    BLTC_CUDA(cudaEventCreate(&e0));
    BLTC_CUDA(cudaEventCreate(&e1));
    k_dfma_loop<<<grid, block>>>(d, 200, 1.0000001, 1e-9);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaEventRecord(e0));
    k_dfma_loop<<<grid, block>>>(d, 2000, 1.0000001, 1e-9);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaEventRecord(e1));
    BLTC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BLTC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // scale to the requested duration, then measure for real
    int iters = (int)(2000.0 * (seconds * 1e3) / (ms > 0.01 ? ms : 0.01));
    if (iters < 2000) iters = 2000;
    BLTC_CUDA(cudaEventRecord(e0));
    k_dfma_loop<<<grid, block>>>(d, iters, 1.0000001, 1e-9);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaEventRecord(e1));
    BLTC_CUDA(cudaEventSynchronize(e1));
    BLTC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *dfma_per_s = (double)grid * block * iters * 16 * 8 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return BLTC_OK;
  } catch (const CudaFailure&) {
    return BLTC_ERR_CUDA;
  }
}

extern "C" BLTC_API int bltc_launch_count(int64_t* out) {
  if (!out) return BLTC_ERR_VALUE;
  *out = (int64_t)bltc::g_launch_count.load();
  return BLTC_OK;
}

extern "C" BLTC_API int bltc_libm_exp_device(int device, int64_t n, const double* x, double* y) {
  using namespace bltc;
  try {
    if (n < 0 || (n > 0 && (!x || !y))) {
      set_error("bltc_libm_exp_device: bad arguments");
      return BLTC_ERR_VALUE;
    }
    if (n == 0) return BLTC_OK;
    if (device >= 0) BLTC_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    BLTC_CUDA(cudaMalloc(&d, 2 * n * sizeof(double)));
    BLTC_CUDA(cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice));
    k_libm_exp<<<(int)((n + 255) / 256), 256>>>(n, d, d + n);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaMemcpy(y, d + n, n * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return BLTC_OK;
  } catch (const CudaFailure&) {
    return BLTC_ERR_CUDA;
  }
}
