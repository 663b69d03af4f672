// Level-synchronous, bit-exact construction of the reference's adaptive
// partition (tree.py:138-253) on the device.
//
// The reference recursion (tree.py:144-177) splits every node at the
// midpoint of its OWN minimal box along the dims whose extent exceeds
// L_max/sqrt(2), drops empty octants, collapses single-child splits and
// reorders particles with a STABLE sort by child code.  Numbering is BFS
// (tree.py:198-217), which is (level, start) order.  Morton keys on a global
// grid cannot reproduce that, so each level is processed as a segmented
// stable partition:
//
//   k_decide      one thread per node of the level: leaf / ZeroExtent /
//                 split dims + midpoint (exact IEEE ops, no FMA)
//   k_code        one CTA per 2048-element tile: 3-bit child code per element,
//                 per-tile code histogram
//   k_scan_tiles  exclusive scan of the histograms over tiles, per code
//   k_node_counts one warp per splitting node: per-code counts from the tile
//                 prefix (G_c at node start/stop), drop nodes with < 2
//                 non-empty children (tree.py:163-167)
//   scan          child numbering: children of level-L nodes, in node order,
//                 then code order == BFS order
//   k_scatter     stable scatter: dest = start + off[c] + (G_c(i) - G_c(start))
//   k_box         per-child minimal boxes (order-independent min/max, exact)
//
// Data: SoA float64 x,y,z[,q] + int32 original index, ping-ponged per level.
#include <algorithm>

#include "bltc_internal.cuh"

namespace bltc {

namespace {
constexpr int kTileThreads = 256;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;   // 2048
constexpr int kNoCode = 8;
constexpr double kSqrt2 = 1.4142135623730951;       // math.sqrt(2.0) (tree.py:29)

__device__ __forceinline__ unsigned long long d2ord(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord2d(unsigned long long u) {
  u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double((long long)u);
}

__global__ void k_init_boxes(unsigned long long* box_u, int64_t begin, int64_t end) {
  int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= end) return;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    box_u[i * 6 + d] = ~0ull;      // min accumulator
    box_u[i * 6 + 3 + d] = 0ull;   // max accumulator
  }
}

// Minimal bounding boxes (tree.py:138-141): exact min/max via order-preserving
// integer atomics.  After the level's scatter the particles of every node are
// contiguous, so each warp walks a contiguous chunk of kBoxChunk particles
// keeping per-lane running min/max for the node it is in, and reduces and
// flushes them (6 atomics) only when the node changes: one flush per node
// boundary instead of one per 32 particles, which removes the same-address
// atomic contention on large nodes.  Particles in finished leaves carry
// node -1 and are skipped.
constexpr int kBoxChunk = 32 * 16;

__device__ __forceinline__ void box_flush(int nd, unsigned long long (&mn)[3],
                                          unsigned long long (&mx)[3],
                                          unsigned long long* box_u, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn[d], o);
      const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx[d], o);
      mn[d] = a < mn[d] ? a : mn[d];
      mx[d] = b > mx[d] ? b : mx[d];
    }
  }
  if (lane == 0 && nd >= 0 && mx[0] != 0ull) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      atomicMin(&box_u[(int64_t)nd * 6 + d], mn[d]);
      atomicMax(&box_u[(int64_t)nd * 6 + 3 + d], mx[d]);
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    mn[d] = ~0ull;
    mx[d] = 0ull;
  }
}

__global__ void k_box(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                      const double* __restrict__ z, const int32_t* __restrict__ node_of,
                      unsigned long long* box_u) {
  constexpr int kU = 4;                    // 32-particle groups loaded ahead
  constexpr int kNone = -2147483647 - 1;   // past the chunk end
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t c0 = warp * kBoxChunk;
  if (c0 >= n) return;
  const int64_t c1 = min(c0 + kBoxChunk, n);
  unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0ull, 0ull, 0ull};
  int cur = node_of[c0];   // warp-uniform: node being accumulated
  for (int64_t base = c0; base < c1; base += 32 * kU) {
    int ndu[kU];
    unsigned long long vu[kU][3];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + 32 * u + lane;
      ndu[u] = i < c1 ? node_of[i] : kNone;
      vu[u][0] = vu[u][1] = vu[u][2] = 0ull;
      if (i < c1) {
        vu[u][0] = d2ord(x[i]);
        vu[u][1] = d2ord(y[i]);
        vu[u][2] = d2ord(z[i]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool valid = ndu[u] != kNone;
      const int nd = valid ? ndu[u] : cur;
      const unsigned long long* v = vu[u];
      if (valid && nd == cur) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          mn[d] = v[d] < mn[d] ? v[d] : mn[d];
          mx[d] = v[d] > mx[d] ? v[d] : mx[d];
        }
      }
      if (__all_sync(0xffffffffu, nd == cur)) continue;
      // node boundary inside these 32 particles
      box_flush(cur, mn, mx, box_u, lane);
      const int last = __shfl_sync(0xffffffffu, nd, 31);   // invalid lanes hold cur
      if (valid && nd >= 0 && nd != cur && nd != last) {   // nodes wholly inside: rare
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          atomicMin(&box_u[(int64_t)nd * 6 + d], v[d]);
          atomicMax(&box_u[(int64_t)nd * 6 + 3 + d], v[d]);
        }
      }
      if (valid && nd == last && last != cur) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          mn[d] = v[d];
          mx[d] = v[d];
        }
      }
      cur = last;
    }
  }
  box_flush(cur, mn, mx, box_u, lane);
}

__global__ void k_finalize_boxes(const unsigned long long* box_u, double* lo, double* hi,
                                 int64_t begin, int64_t end) {
  int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= end) return;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[i * 3 + d] = ord2d(box_u[i * 6 + d]);
    hi[i * 3 + d] = ord2d(box_u[i * 6 + 3 + d]);
  }
}

// split_dimensions (tree.py:56-67) + leaf tests (tree.py:148-156).
__global__ void k_decide(int64_t begin, int64_t end, const int32_t* __restrict__ start,
                         const int32_t* __restrict__ stop, const double* __restrict__ lo,
                         const double* __restrict__ hi, int64_t max_count, int32_t* split,
                         double* mid) {
  int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = begin + li;
  if (i >= end) return;
  int s = 0;
  if ((int64_t)(stop[i] - start[i]) > max_count) {
    double ext[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) ext[d] = __dsub_rn(hi[i * 3 + d], lo[i * 3 + d]);
    bool zero = ext[0] < kDegenerate && ext[1] < kDegenerate && ext[2] < kDegenerate;
    if (!zero) {
      double emax = ext[0];
      if (ext[1] > emax) emax = ext[1];
      if (ext[2] > emax) emax = ext[2];
      double cutoff = __ddiv_rn(emax, kSqrt2);
      // bit 0 = x, bit 1 = y, bit 2 = z; code bits are emitted x,y,z MSB-first
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (ext[d] > cutoff) s |= 1 << d;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        mid[li * 3 + d] = __dmul_rn(0.5, __dadd_rn(lo[i * 3 + d], hi[i * 3 + d]));
    }
  }
  split[li] = s;
}

__device__ __forceinline__ int child_code(double x, double y, double z, int dims,
                                          const double* m) {
  int c = 0;
  if (dims & 1) c = 2 * c + (x >= m[0]);
  if (dims & 2) c = 2 * c + (y >= m[1]);
  if (dims & 4) c = 2 * c + (z >= m[2]);
  return c;
}

__global__ void __launch_bounds__(kTileThreads)
k_code(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
       const double* __restrict__ z, const int32_t* __restrict__ node_of, int64_t begin,
       int64_t end, const int32_t* __restrict__ split, const double* __restrict__ mid,
       uint8_t* __restrict__ code, int32_t* __restrict__ tile_cnt) {
  __shared__ int cnt[8];
  if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int64_t tile0 = (int64_t)blockIdx.x * kTile;
  int local[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int r = 0; r < kTileItems; ++r) {
    int64_t i = tile0 + r * kTileThreads + threadIdx.x;
    int c = kNoCode;
    if (i < n) {
      int nd = node_of[i];
      if (nd >= begin && nd < end) {
        int li = nd - (int)begin;
        int dims = split[li];
        if (dims) c = child_code(x[i], y[i], z[i], dims, mid + li * 3);
      }
      code[i] = (uint8_t)c;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) local[k] += __popc(__ballot_sync(0xffffffffu, c == k));
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (local[k]) atomicAdd(&cnt[k], local[k]);
  }
  __syncthreads();
  if (threadIdx.x < 8) tile_cnt[blockIdx.x * 8 + threadIdx.x] = cnt[threadIdx.x];
}

// In-place exclusive scan over tiles, one warp per code; writes the grand
// total at index ntiles.
__global__ void k_scan_tiles(int32_t* tile_cnt, int64_t ntiles) {
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  int carry = 0;
  for (int64_t t0 = 0; t0 < ntiles; t0 += 32) {
    int64_t t = t0 + lane;
    int v = t < ntiles ? tile_cnt[t * 8 + c] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (t < ntiles) tile_cnt[t * 8 + c] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) tile_cnt[ntiles * 8 + c] = carry;
}

// G_c(p) for all 8 codes: elements with code c before position p.
__device__ __forceinline__ void warp_prefix_at(int64_t p, int64_t n, const uint8_t* code,
                                               const int32_t* tile_cnt, int out[8]) {
  const int lane = threadIdx.x & 31;
  int64_t t = p / kTile;
  int64_t t0 = t * kTile;
  int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = t0 + lane; i < p; i += 32) {
    int c = code[i];
#pragma unroll
    for (int k = 0; k < 8; ++k) cnt[k] += (c == k);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int v = cnt[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    out[k] = tile_cnt[t * 8 + k] + v;
  }
}

__global__ void k_node_counts(int64_t n, int64_t begin, int64_t end,
                              const int32_t* __restrict__ start, const int32_t* __restrict__ stop,
                              int32_t* split, const uint8_t* __restrict__ code,
                              const int32_t* __restrict__ tile_cnt, int32_t* node_base,
                              int32_t* node_off, int32_t* node_nchild) {
  int64_t li = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (begin + li >= end) return;
  int64_t i = begin + li;
  if (split[li] == 0) {
    if (lane == 0) node_nchild[li] = 0;
    return;
  }
  int g0[8], g1[8];
  warp_prefix_at(start[i], n, code, tile_cnt, g0);
  warp_prefix_at(stop[i], n, code, tile_cnt, g1);
  if (lane == 0) {
    int nonempty = 0, off = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int c = g1[k] - g0[k];
      nonempty += c > 0;
      node_base[li * 8 + k] = g0[k];
      node_off[li * 8 + k] = off;
      off += c;
    }
    if (nonempty < 2) {   // tree.py:163-167: trivial split collapses into a leaf
      split[li] = 0;
      nonempty = 0;
    }
    node_nchild[li] = nonempty;
  }
}

__global__ void k_make_children(int64_t begin, int64_t end, int64_t level_end,
                                const int32_t* __restrict__ split,
                                const int32_t* __restrict__ nchild,
                                const int32_t* __restrict__ child_prefix,
                                const int32_t* __restrict__ node_off, int32_t* start,
                                int32_t* stop, int32_t* child_start, int32_t* child_count,
                                int32_t* level, int32_t* node_child) {
  int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = begin + li;
  if (i >= end) return;
  int nc = nchild[li];
  if (nc == 0 || split[li] == 0) {
    child_start[i] = -1;
    child_count[i] = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) node_child[li * 8 + k] = -1;
    return;
  }
  int first = (int)level_end + child_prefix[li];
  child_start[i] = first;
  child_count[i] = nc;
  int s0 = start[i], lv = level[i] + 1, j = 0;
  int total = stop[i] - s0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int o = node_off[li * 8 + k];
    int o1 = k < 7 ? node_off[li * 8 + k + 1] : total;
    int cnt = o1 - o;
    if (cnt > 0) {
      int id = first + j++;
      start[id] = s0 + o;
      stop[id] = s0 + o + cnt;
      level[id] = lv;
      child_start[id] = -1;
      child_count[id] = 0;
      node_child[li * 8 + k] = id;
    } else {
      node_child[li * 8 + k] = -1;
    }
  }
}

// Stable scatter of one level.  Per tile, the rank of an element among the
// tile's elements with the same code is reconstructed exactly as k_code
// counted them (round-major, warp, lane == ascending index).
__global__ void __launch_bounds__(kTileThreads)
k_scatter(int64_t n, int64_t begin, const double* __restrict__ x0, const double* __restrict__ y0,
          const double* __restrict__ z0, const double* __restrict__ q0,
          const int32_t* __restrict__ o0, const int32_t* __restrict__ node_of0,
          const uint8_t* __restrict__ code, const int32_t* __restrict__ tile_cnt,
          const int32_t* __restrict__ split, const int32_t* __restrict__ start,
          const int32_t* __restrict__ node_base, const int32_t* __restrict__ node_off,
          const int32_t* __restrict__ node_child, double* __restrict__ x1,
          double* __restrict__ y1, double* __restrict__ z1, double* __restrict__ q1,
          int32_t* __restrict__ o1, int32_t* __restrict__ node_of1) {
  __shared__ int wcnt[kTileItems][kTileThreads / 32][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int64_t tile0 = (int64_t)blockIdx.x * kTile;
  int my_code[kTileItems], my_rank[kTileItems];
#pragma unroll
  for (int r = 0; r < kTileItems; ++r) {
    int64_t i = tile0 + r * kTileThreads + threadIdx.x;
    int c = i < n ? code[i] : kNoCode;
    my_code[r] = c;
    my_rank[r] = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      unsigned b = __ballot_sync(0xffffffffu, c == k);
      if (c == k) my_rank[r] = __popc(b & lt);
      if (lane == 0) wcnt[r][warp][k] = __popc(b);
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) {   // exclusive prefix over (round, warp) per code
    int k = threadIdx.x, acc = 0;
    for (int r = 0; r < kTileItems; ++r)
      for (int w = 0; w < kTileThreads / 32; ++w) {
        int v = wcnt[r][w][k];
        wcnt[r][w][k] = acc;
        acc += v;
      }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kTileItems; ++r) {
    int64_t i = tile0 + r * kTileThreads + threadIdx.x;
    if (i >= n) continue;
    int c = my_code[r];
    int64_t dest = i;
    int new_node = -1;
    if (c != kNoCode) {
      int nd = node_of0[i];
      int li = nd - (int)begin;
      if (split[li]) {
        int g = tile_cnt[blockIdx.x * 8 + c] + wcnt[r][warp][c] + my_rank[r];
        dest = (int64_t)start[nd] + node_off[li * 8 + c] + (g - node_base[li * 8 + c]);
        new_node = node_child[li * 8 + c];
      }
    }
    x1[dest] = x0[i];
    y1[dest] = y0[i];
    z1[dest] = z0[i];
    if (q0) q1[dest] = q0[i];
    o1[dest] = o0[i];
    node_of1[dest] = new_node;
  }
}

__global__ void k_iota(int32_t* o, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) o[i] = (int32_t)i;
}

__global__ void k_perm(const int32_t* order, int32_t* perm, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) perm[order[i]] = (int32_t)i;
}

__global__ void k_root(int32_t* start, int32_t* stop, int32_t* level, int64_t n) {
  start[0] = 0;
  stop[0] = (int32_t)n;
  level[0] = 0;
}

__global__ void k_leaf_flags(int64_t nn, const int32_t* start, const int32_t* child_count,
                             int32_t* flag_at_start, int32_t* node_at_start) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (child_count[i] == 0) {
    flag_at_start[start[i]] = 1;
    node_at_start[start[i]] = (int32_t)i;
  }
}

__global__ void k_leaf_compact(int64_t n, const int32_t* flag, const int32_t* pos,
                               const int32_t* node_at_start, int32_t* leaves) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && flag[i]) leaves[pos[i]] = node_at_start[i];
}

inline int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, g);
}
}  // namespace

void build_partition(Partition& P, BuildScratch& S, int64_t n, const double* dx,
                     const double* dy, const double* dz, const double* dq, int64_t max_count,
                     cudaStream_t st, HostScratch& hs) {
  P.n = n;
  const bool with_q = dq != nullptr;
  P.x.resize(n); P.y.resize(n); P.z.resize(n); P.order.resize(n); P.perm.resize(n);
  if (with_q) P.q.resize(n);
  S.x1.resize(n); S.y1.resize(n); S.z1.resize(n); S.o1.resize(n);
  if (with_q) S.q1.resize(n);
  S.node_of0.resize(n); S.node_of1.resize(n); S.code.resize(n);
  const int64_t ntiles = (n + kTile - 1) / kTile;
  S.tile_cnt.resize((ntiles + 1) * 8);

  // buffers: cur = P.*, nxt = S.*; swapped by pointer each level.
  double *cx = P.x.p, *cy = P.y.p, *cz = P.z.p, *cq = with_q ? P.q.p : nullptr;
  double *nx = S.x1.p, *ny = S.y1.p, *nz = S.z1.p, *nq = with_q ? S.q1.p : nullptr;
  int32_t *co = P.order.p, *no = S.o1.p, *cn = S.node_of0.p, *nn_ = S.node_of1.p;
  BLTC_CUDA(cudaMemcpyAsync(cx, dx, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  BLTC_CUDA(cudaMemcpyAsync(cy, dy, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  BLTC_CUDA(cudaMemcpyAsync(cz, dz, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (with_q) BLTC_CUDA(cudaMemcpyAsync(cq, dq, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  k_iota<<<grid_for(n, 256), 256, 0, st>>>(co, n);
  BLTC_LAUNCH_CHECK();
  BLTC_CUDA(cudaMemsetAsync(cn, 0, n * sizeof(int32_t), st));

  // node storage (grown as levels are added)
  int64_t cap = std::max<int64_t>(1024, 2 * n / std::max<int64_t>(1, max_count) + 64);
  auto ensure_nodes = [&](int64_t need) {
    const int64_t c = need;
    P.start.n = P.stop.n = P.child_start.n = P.child_count.n = P.level.n = P.n_nodes;
    P.lo.n = P.hi.n = P.n_nodes * 3;
    S.box_u.n = P.n_nodes * 6;
    P.start.grow_keep(c, st); P.stop.grow_keep(c, st); P.child_start.grow_keep(c, st);
    P.child_count.grow_keep(c, st); P.level.grow_keep(c, st);
    P.lo.grow_keep(3 * c, st); P.hi.grow_keep(3 * c, st);
    S.box_u.grow_keep(6 * c, st);
  };
  P.n_nodes = 0;
  ensure_nodes(cap);
  P.n_nodes = 1;
  k_root<<<1, 1, 0, st>>>(P.start.p, P.stop.p, P.level.p, n);
  BLTC_LAUNCH_CHECK();
  k_init_boxes<<<1, 32, 0, st>>>(S.box_u.p, 0, 1);
  BLTC_LAUNCH_CHECK();
  k_box<<<grid_for((n + kBoxChunk - 1) / kBoxChunk * 32, 256), 256, 0, st>>>(n, cx, cy, cz, cn,
                                                                          S.box_u.p);
  BLTC_LAUNCH_CHECK();
  k_finalize_boxes<<<1, 32, 0, st>>>(S.box_u.p, P.lo.p, P.hi.p, 0, 1);
  BLTC_LAUNCH_CHECK();

  P.level_begin.assign(1, 0);
  int64_t begin = 0, end = 1;
  int32_t depth = 0;
  int32_t* hbuf = (int32_t*)hs.get(64);
  while (true) {
    const int64_t nl = end - begin;
    S.node_split.resize(nl); S.node_mid.resize(nl * 3); S.node_base.resize(nl * 8);
    S.node_off.resize(nl * 8); S.node_child.resize(nl * 8); S.node_nchild.resize(nl + 1);
    S.counter.resize(nl + 1);
    k_decide<<<grid_for(nl, 128), 128, 0, st>>>(begin, end, P.start.p, P.stop.p, P.lo.p,
                                                  P.hi.p, max_count, S.node_split.p,
                                                  S.node_mid.p);
    BLTC_LAUNCH_CHECK();
    k_code<<<(int)ntiles, kTileThreads, 0, st>>>(n, cx, cy, cz, cn, begin, end, S.node_split.p,
                                                 S.node_mid.p, S.code.p, S.tile_cnt.p);
    BLTC_LAUNCH_CHECK();
    k_scan_tiles<<<1, 256, 0, st>>>(S.tile_cnt.p, ntiles);
    BLTC_LAUNCH_CHECK();
    k_node_counts<<<grid_for(nl * 32, 256), 256, 0, st>>>(
        n, begin, end, P.start.p, P.stop.p, S.node_split.p, S.code.p, S.tile_cnt.p,
        S.node_base.p, S.node_off.p, S.node_nchild.p);
    BLTC_LAUNCH_CHECK();
    BLTC_CUDA(cudaMemsetAsync(S.node_nchild.p + nl, 0, sizeof(int32_t), st));
    exclusive_scan_i32(S.node_nchild.p, S.counter.p, nl + 1, S.scan_tmp, st);
    BLTC_CUDA(cudaMemcpyAsync(hbuf, S.counter.p + nl, sizeof(int32_t), cudaMemcpyDeviceToHost,
                              st));
    BLTC_CUDA(cudaStreamSynchronize(st));
    const int64_t total_children = hbuf[0];
    ensure_nodes(end + total_children);
    k_make_children<<<grid_for(nl, 128), 128, 0, st>>>(
        begin, end, end, S.node_split.p, S.node_nchild.p, S.counter.p, S.node_off.p, P.start.p,
        P.stop.p, P.child_start.p, P.child_count.p, P.level.p, S.node_child.p);
    BLTC_LAUNCH_CHECK();
    if (total_children == 0) break;
    k_scatter<<<(int)ntiles, kTileThreads, 0, st>>>(
        n, begin, cx, cy, cz, cq, co, cn, S.code.p, S.tile_cnt.p, S.node_split.p, P.start.p,
        S.node_base.p, S.node_off.p, S.node_child.p, nx, ny, nz, nq, no, nn_);
    BLTC_LAUNCH_CHECK();
    std::swap(cx, nx); std::swap(cy, ny); std::swap(cz, nz); std::swap(cq, nq);
    std::swap(co, no); std::swap(cn, nn_);
    const int64_t nb = end, ne = end + total_children;
    k_init_boxes<<<grid_for(ne - nb, 128), 128, 0, st>>>(S.box_u.p, nb, ne);
    BLTC_LAUNCH_CHECK();
    k_box<<<grid_for((n + kBoxChunk - 1) / kBoxChunk * 32, 256), 256, 0, st>>>(n, cx, cy, cz, cn,
                                                                          S.box_u.p);
    BLTC_LAUNCH_CHECK();
    k_finalize_boxes<<<grid_for(ne - nb, 128), 128, 0, st>>>(S.box_u.p, P.lo.p, P.hi.p, nb, ne);
    BLTC_LAUNCH_CHECK();
    P.n_nodes = ne;
    P.level_begin.push_back(nb);
    begin = nb;
    end = ne;
    ++depth;
  }
  P.level_begin.push_back(end);
  P.depth = depth;
  // Final arrays must live in P.*: copy back if the last level left them in S.*.
  if (cx != P.x.p) {
    BLTC_CUDA(cudaMemcpyAsync(P.x.p, cx, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BLTC_CUDA(cudaMemcpyAsync(P.y.p, cy, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BLTC_CUDA(cudaMemcpyAsync(P.z.p, cz, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (with_q)
      BLTC_CUDA(cudaMemcpyAsync(P.q.p, cq, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BLTC_CUDA(cudaMemcpyAsync(P.order.p, co, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  }
  k_perm<<<grid_for(n, 256), 256, 0, st>>>(P.order.p, P.perm.p, n);
  BLTC_LAUNCH_CHECK();
  P.start.n = P.stop.n = P.child_start.n = P.child_count.n = P.level.n = P.n_nodes;
  P.lo.n = P.hi.n = 3 * P.n_nodes;
}

void partition_leaves(Partition& P, BuildScratch& S, cudaStream_t st, HostScratch& hs) {
  const int64_t n = P.n;
  S.node_of0.resize(n);   // flags
  S.node_of1.resize(n);   // node at start
  S.o1.resize(n);         // scanned positions
  BLTC_CUDA(cudaMemsetAsync(S.node_of0.p, 0, n * sizeof(int32_t), st));
  k_leaf_flags<<<grid_for(P.n_nodes, 256), 256, 0, st>>>(P.n_nodes, P.start.p, P.child_count.p,
                                                         S.node_of0.p, S.node_of1.p);
  BLTC_LAUNCH_CHECK();
  exclusive_scan_i32(S.node_of0.p, S.o1.p, n, S.scan_tmp, st);
  int32_t* h = (int32_t*)hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, S.o1.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaMemcpyAsync(h + 1, S.node_of0.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  P.n_leaves = h[0] + h[1];
  P.leaves.resize(P.n_leaves);
  k_leaf_compact<<<grid_for(n, 256), 256, 0, st>>>(n, S.node_of0.p, S.o1.p, S.node_of1.p,
                                                   P.leaves.p);
  BLTC_LAUNCH_CHECK();
}

}  // namespace bltc
