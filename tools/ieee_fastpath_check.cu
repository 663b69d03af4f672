// Bitwise check of eval_common.cuh's sqrt_rn_fastpath / div_rn_fastpath
// against __dsqrt_rn / __ddiv_rn wherever the fast-path test holds, over
// random operands spanning many binades.  Prints mismatch and coverage counts.
#include <cstdio>
#include "../paper_2003_01836_b200/csrc/eval_common.cuh"
using namespace bltc;
__device__ unsigned long long g_cnt[6];
__device__ double g_bad[16];
__global__ void k(long n, unsigned long long seed) {
  unsigned long long mism = 0, okc = 0, mism_d = 0, okd = 0, okr = 0, mism_r = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    unsigned long long h2 = h * 0x94D049BB133111EBull; h2 ^= h2 >> 32;
    const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    const double v = (double)(h2 >> 11) * (1.0 / 9007199254740992.0);
    const double x = exp2(-200.0 + 400.0 * u);
    const double a = (v - 0.5) * exp2(-60.0 + 120.0 * u);
    bool ok;
    const double s = sqrt_rn_fastpath(x, ok);
    if (ok) { ++okc; if (__double_as_longlong(s) != __double_as_longlong(__dsqrt_rn(x))) ++mism; }
    const double q = div_rn_fastpath(a, s, ok);
    if (ok) { ++okd; if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, s))) ++mism_d; }
    const double rb = (v - 0.5) * exp2(-1100.0 + 2200.0 * u);   // across the whole range
    const double r = rcp_rn_fastpath(rb, ok);
    if (ok) {
      ++okr;
      if (__double_as_longlong(r) != __double_as_longlong(__drcp_rn(rb))) {
        ++mism_r;
        const unsigned long long k = atomicAdd(&g_cnt[5], 0ull);
        if (k < 16) g_bad[k] = rb;
      }
    }
  }
  atomicAdd(&g_cnt[4], okr); atomicAdd(&g_cnt[5], mism_r);
  atomicAdd(&g_cnt[0], okc); atomicAdd(&g_cnt[1], mism); atomicAdd(&g_cnt[2], okd); atomicAdd(&g_cnt[3], mism_d);
}
int main() {
  k<<<148 * 8, 256>>>(1L << 32, 777);
  unsigned long long h[6]; cudaMemcpyFromSymbol(h, g_cnt, sizeof(h));
  printf("{\"sqrt_fastpath\": %llu, \"sqrt_mismatch\": %llu, \"div_fastpath\": %llu, \"div_mismatch\": %llu, \"rcp_fastpath\": %llu, \"rcp_mismatch\": %llu}\n", h[0], h[1], h[2], h[3], h[4], h[5]);
  double bad[16]; cudaMemcpyFromSymbol(bad, g_bad, sizeof(bad));
  for (int i = 0; i < 16; ++i) printf("rcp mismatch operand %a\n", bad[i]);
  return 0;
}
