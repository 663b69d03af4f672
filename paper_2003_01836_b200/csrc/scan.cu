// Device-wide exclusive prefix sum (int32), used for CSR construction and
// stream compaction.  Three-phase: per-block totals -> scan of totals
// (recursive) -> per-block scan plus carried offset.
#include <algorithm>

#include "bltc_internal.cuh"

namespace bltc {

namespace {
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns block total.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
    int wi = warp_incl_scan(w);
    if (lane < kScanThreads / 32) warp_sums[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  int r = inc - v + warp_sums[warp];
  __syncthreads();
  return r;
}

__global__ void k_block_totals(const int32_t* in, int64_t n, int32_t* totals) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  __shared__ int tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) totals[blockIdx.x] = tot;
}

__global__ void k_block_scan(const int32_t* in, int32_t* out, int64_t n, const int32_t* offsets) {
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  __shared__ int tot;
  int pre = block_excl_scan(s, &tot) + (offsets ? offsets[blockIdx.x] : 0);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    if (i < n) out[i] = pre;
    pre += v[k];
  }
}
}  // namespace

int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

static size_t scan_tmp_need(int64_t n) {
  if (n <= kScanTile) return 0;
  int64_t nblk = ceil_div(n, kScanTile);
  return 2 * (size_t)nblk + scan_tmp_need(nblk);
}

static void scan_rec(const int32_t* in, int32_t* out, int64_t n, int32_t* tmp, cudaStream_t st) {
  int nblk = ceil_div(n, kScanTile);
  if (nblk == 1) {
    k_block_scan<<<1, kScanThreads, 0, st>>>(in, out, n, nullptr);
    BLTC_LAUNCH_CHECK();
    return;
  }
  int32_t* totals = tmp;
  int32_t* offsets = tmp + nblk;
  k_block_totals<<<nblk, kScanThreads, 0, st>>>(in, n, totals);
  BLTC_LAUNCH_CHECK();
  scan_rec(totals, offsets, nblk, tmp + 2 * (size_t)nblk, st);
  k_block_scan<<<nblk, kScanThreads, 0, st>>>(in, out, n, offsets);
  BLTC_LAUNCH_CHECK();
}

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, DBuf<int32_t>& tmp,
                        cudaStream_t st) {
  if (n <= 0) return;
  size_t need = scan_tmp_need(n);
  if (need > tmp.cap) {
    BLTC_CUDA(cudaStreamSynchronize(st));
    tmp.reserve(need);
  }
  scan_rec(in, out, n, tmp.p, st);
}

namespace {
__global__ void k_sum_i64(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                          int64_t n, unsigned long long* out) {
  unsigned long long sa = 0, sb = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    sa += (unsigned long long)(unsigned)a[i];
    sb += (unsigned long long)(unsigned)b[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, sa);
    atomicAdd(out + 1, sb);
  }
}
}  // namespace

void sum_counts_i64(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* out,
                    cudaStream_t st) {
  BLTC_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), st));
  if (n <= 0) return;
  int grid = (int)std::min<int64_t>((n + 255) / 256, 1184);
  k_sum_i64<<<grid, 256, 0, st>>>(a, b, n, out);
  BLTC_LAUNCH_CHECK();
}

}  // namespace bltc
