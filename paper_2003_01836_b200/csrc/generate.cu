// On-device input generation: the reference harness's
// uniform particles (cli.py:54-62) -- numpy Generator(Philox(child)).uniform
// -- reproduced bit for bit on the GPU.
//
// numpy's Philox is Philox4x64-10 (Random123): the 256-bit counter is
// incremented BEFORE each block of four 64-bit outputs, which are consumed
// in order; uniform(low, high) = low + (high - low) * ((u >> 11) * 2^-53).
// The key and the starting counter come from numpy on the host
// (Philox(SeedSequence child).state), so the seed-sequence hashing stays in
// numpy.  One thread per 4-draw block; draw j of an array of `dims`
// interleaved components (row-major (n, dims) as numpy fills it) lands in
// component j % dims, element j / dims.
#include "bltc_internal.cuh"

namespace bltc {
namespace {

__device__ __forceinline__ void philox4x64_10(unsigned long long (&c)[4], unsigned long long k0,
                                              unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

struct Out4 {
  double* p[4];
};

__global__ void k_philox_uniform(unsigned long long k0, unsigned long long k1,
                                 unsigned long long c0, unsigned long long c1,
                                 unsigned long long c2, unsigned long long c3, int64_t n,
                                 int dims, double low, double span, Out4 out) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = n * dims;
  if (4 * b >= total) return;
  // counter + 1 + b, 256-bit
  unsigned long long c[4] = {c0, c1, c2, c3};
  const unsigned long long add = (unsigned long long)b + 1ull;
  const unsigned long long s0 = c[0] + add;
  unsigned long long carry = s0 < c[0] ? 1ull : 0ull;
  c[0] = s0;
  for (int w = 1; w < 4 && carry; ++w) {
    c[w] += 1ull;
    carry = c[w] == 0ull ? 1ull : 0ull;
  }
  philox4x64_10(c, k0, k1);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int64_t j = 4 * b + w;
    if (j < total) {
      const double u = (double)(c[w] >> 11) * (1.0 / 9007199254740992.0);
      out.p[j % dims][j / dims] = __dadd_rn(low, __dmul_rn(span, u));
    }
  }
}

}  // namespace
}  // namespace bltc

extern "C" BLTC_API int bltc_philox_uniform(int device, const uint64_t* key,
                                            const uint64_t* counter, int64_t n, int32_t dims,
                                            double low, double high, double* const* out) {
  using namespace bltc;
  try {
    if (!key || !counter || !out || n < 0 || dims < 1 || dims > 4) {
      set_error("bltc_philox_uniform: invalid arguments");
      return BLTC_ERR_VALUE;
    }
    if (device >= 0) BLTC_CUDA(cudaSetDevice(device));
    if (n == 0) return BLTC_OK;
    Out4 o{};
    for (int d = 0; d < dims; ++d) o.p[d] = out[d];
    const int64_t blocks = (n * dims + 3) / 4;
    k_philox_uniform<<<(unsigned)((blocks + 255) / 256), 256>>>(
        key[0], key[1], counter[0], counter[1], counter[2], counter[3], n, dims, low,
        high - low, o);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaDeviceSynchronize());
    return BLTC_OK;
  } catch (const CudaFailure&) {
    return BLTC_ERR_CUDA;
  }
}
