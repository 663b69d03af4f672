// Batch x cluster interaction lists (engine.py:65-130) as flat CSR.
//
// One thread per target batch walks the cluster tree depth-first with an
// explicit stack, applying the reference MAC (engine.py:74-85) with its
// exact operation order (no FMA, IEEE sqrt):
//   accept            -> approx list
//   SIZE failure      -> direct list, no recursion
//   GEOMETRY failure  -> leaf ? direct : recurse into the children in order
// The DFS visit order makes every list ascending in cluster start, exactly
// the reference's list order.  Two passes (count, then fill after a scan)
// emit CSR with one segment per (batch, source group); entries are global
// cluster ids (group cluster offset + local BFS id).
#include "bltc_internal.cuh"

namespace bltc {

namespace {
constexpr int kStack = 512;

__device__ __forceinline__ bool mac_geometry_ok(double bx, double by, double bz, double br,
                                                const MacNode& c, double theta) {
  double dx = __dsub_rn(bx, c.cx);
  double dy = __dsub_rn(by, c.cy);
  double dz = __dsub_rn(bz, c.cz);
  double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                     __dmul_rn(dz, dz)));
  return __dadd_rn(br, c.radius) < __dmul_rn(theta, dist);
}
}  // namespace

// fill == false: count entries, accumulate pair counts.  fill == true: write.
__global__ void k_lists(int64_t nb, int G, int g, const double* __restrict__ bcenter,
                        const double* __restrict__ bradius, const int32_t* __restrict__ bstart,
                        const int32_t* __restrict__ bstop, const MacNode* __restrict__ nodes,
                        int32_t cluster_offset, double theta, int64_t per_node, bool fill,
                        int32_t* __restrict__ a_cnt, int32_t* __restrict__ d_cnt,
                        const int32_t* __restrict__ a_ptr, const int32_t* __restrict__ d_ptr,
                        int32_t* __restrict__ a_idx, int32_t* __restrict__ d_idx,
                        unsigned long long* pairs, int32_t* overflow) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const double bx = bcenter[3 * b], by = bcenter[3 * b + 1], bz = bcenter[3 * b + 2];
  const double br = bradius[b];
  int stack[kStack];
  int sp = 0;
  stack[sp++] = 0;
  int na = 0, nd = 0;
  long long dcount = 0;
  int32_t* ap = nullptr;
  int32_t* dp = nullptr;
  if (fill) {
    ap = a_idx + a_ptr[b * G + g];
    dp = d_idx + d_ptr[b * G + g];
  }
  while (sp > 0) {
    const int ci = stack[--sp];
    const MacNode c = nodes[ci];
    bool geom = mac_geometry_ok(bx, by, bz, br, c, theta);
    if (geom && c.eligible) {
      if (per_node < (int64_t)c.count) {          // accepted
        if (fill) ap[na] = cluster_offset + ci;
        ++na;
        continue;
      }
      if (fill) dp[nd] = cluster_offset + ci;     // SIZE failure
      ++nd;
      dcount += c.count;
      continue;
    }
    if (c.child_count == 0) {                     // GEOMETRY failure at a leaf
      if (fill) dp[nd] = cluster_offset + ci;
      ++nd;
      dcount += c.count;
      continue;
    }
    if (sp + c.child_count > kStack) {
      atomicExch(overflow, 1);
      return;
    }
    for (int k = c.child_count - 1; k >= 0; --k) stack[sp++] = c.child_start + k;
  }
  if (!fill) {
    a_cnt[b * G + g] = na;
    d_cnt[b * G + g] = nd;
    long long nt = bstop[b] - bstart[b];
    atomicAdd(&pairs[0], (unsigned long long)(nt * dcount));
    atomicAdd(&pairs[1], (unsigned long long)(nt * per_node * na));
  }
}

__global__ void k_mark_used(int64_t n, const int32_t* __restrict__ idx, int32_t* used) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) used[idx[i]] = 1;
}

}  // namespace bltc
