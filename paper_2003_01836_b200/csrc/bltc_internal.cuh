// Internal definitions shared by the libbltc translation units.
//
// Device data model (one "source group" = one rank's source tree; a single
// device run has exactly one group):
//   * particles: SoA float64 x,y,z,q, reordered cluster-contiguously
//     (tree.py:219-221 semantics: order = reordered -> original, perm = inverse)
//   * clusters: BFS-numbered (tree.py:198-217), children contiguous
//   * lists: CSR over target batches, entries are global cluster ids in the
//     reference DFS order (engine.py:96-125)
//   * moments: (n+1)^3 rows, k1-major (moments.py:24-25)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/bltc.h"

namespace bltc {

constexpr double kSingularSq = 1e-28;                     // kernels.py:25
constexpr double kNodeTol = 2.2250738585072014e-308;      // interp.py:28
constexpr double kDegenerate = 1e-14;                     // tree.py:30
constexpr int kMaxDegree = 20;                            // supported interpolation degree
constexpr int kMaxM = kMaxDegree + 1;

// Packed record used by the MAC walk (48 bytes, one load per visited node).
struct __align__(16) MacNode {
  double cx, cy, cz, radius;
  int32_t count;
  int32_t child_start;   // BFS id of first child (-1 for leaves)
  int32_t child_count;
  int32_t eligible;
};

// Cluster geometry/ranges used by the evaluation kernels.
struct __align__(16) EvalCluster {
  double lo[3];
  double hi[3];
  int32_t start, stop;   // particle range in the group's concatenated arrays
  int32_t mrow;          // moment row (-1: none)
  int32_t pad;
};

void set_error(const std::string& msg);

#define BLTC_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::bltc::set_error(std::string(#call) + ": " + cudaGetErrorString(_e) +   \
                        " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
      throw ::bltc::CudaFailure();                                             \
    }                                                                          \
  } while (0)

// Every kernel launch is followed by exactly one BLTC_LAUNCH_CHECK(): it
// checks the launch and counts it -- process-wide (atomic: rank threads of
// bltc_run_distributed launch concurrently; bltc_launch_count) and per host
// thread (bltc_stats.kernel_launches of that thread's calls).
extern std::atomic<long long> g_launch_count;
extern thread_local long long t_launch_count;
#define BLTC_LAUNCH_CHECK()                                          \
  do {                                                               \
    BLTC_CUDA(cudaGetLastError());                                   \
    ::bltc::g_launch_count.fetch_add(1, std::memory_order_relaxed); \
    ++::bltc::t_launch_count;                                        \
  } while (0)

struct CudaFailure {};
struct UserError {
  int code;
};

// Grow-only device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  size_t n = 0;
  void reserve(size_t count) {
    if (count <= cap) return;
    if (p) BLTC_CUDA(cudaFree(p));
    p = nullptr;
    size_t c = count < 16 ? 16 : count;
    BLTC_CUDA(cudaMalloc(&p, c * sizeof(T)));
    cap = c;
  }
  void resize(size_t count) {
    reserve(count);
    n = count;
  }
  // Grow to hold at least `count` elements, keeping the first min(n, cap).
  // Each buffer checks its own capacity: buffers shared between partitions
  // (BuildScratch) must not rely on another buffer's capacity as a proxy.
  void grow_keep(size_t count, cudaStream_t s) {
    if (count <= cap) return;
    T* q = nullptr;
    size_t c = count + count / 2;
    if (c < 2 * cap) c = 2 * cap;
    BLTC_CUDA(cudaMalloc(&q, c * sizeof(T)));
    const size_t keep = n < cap ? n : cap;
    if (p && keep)
      BLTC_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) {
      BLTC_CUDA(cudaStreamSynchronize(s));
      BLTC_CUDA(cudaFree(p));
    }
    p = q;
    cap = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = n = 0;
  }
};

// Pinned host scratch for small readbacks.
// An auxiliary stream with fork / join events (the bitwise upward pass runs
// the big clusters' split items on it, concurrent with the small clusters).
struct BwStreams {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

struct HostScratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      BLTC_CUDA(cudaMallocHost(&p, bytes));
      cap = bytes;
    }
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// ---------------------------------------------------------------------------
// Partition (tree / batch) builder: tree.py:138-253 on the device.
struct Partition {
  int64_t n = 0;
  int64_t n_nodes = 0;
  int32_t depth = 0;
  // reordered particles (x,y,z[,q]) and reordered -> original index
  DBuf<double> x, y, z, q;
  DBuf<int32_t> order;
  DBuf<int32_t> perm;   // original -> reordered
  // BFS nodes
  DBuf<int32_t> start, stop, child_start, child_count, level;
  DBuf<double> lo, hi;  // [node*3 + d]
  // leaves sorted by start (== DFS leaf order, tree.py:240-250)
  int64_t n_leaves = 0;
  DBuf<int32_t> leaves;
  std::vector<int64_t> level_begin;  // host copy: node id range per level
};

struct BuildScratch {
  DBuf<double> x1, y1, z1, q1;
  DBuf<int32_t> o1, node_of0, node_of1;
  DBuf<uint8_t> code;
  DBuf<int32_t> tile_cnt;       // [tiles+1][8]
  DBuf<int32_t> node_base;      // [level nodes][8] G_c(start)
  DBuf<int32_t> node_off;       // [level nodes][8] child offsets within node
  DBuf<int32_t> node_child;     // [level nodes][8] child id per code (-1)
  DBuf<int32_t> node_nchild;    // [level nodes]
  DBuf<int32_t> node_split;     // [level nodes] tentative split: dims mask (0: no)
  DBuf<double> node_mid;        // [level nodes][3]
  DBuf<unsigned long long> box_u;  // [node][6] ordered-int min/max accumulation
  DBuf<int32_t> scan_tmp;
  DBuf<int32_t> counter;
};

void build_partition(Partition& P, BuildScratch& S, int64_t n, const double* dx,
                     const double* dy, const double* dz, const double* dq, int64_t max_count,
                     cudaStream_t st, HostScratch& hs);
void partition_leaves(Partition& P, BuildScratch& S, cudaStream_t st, HostScratch& hs);

// Geometry derived from boxes (tree.py:46-53, 206).
void make_mac_nodes(const Partition& P, DBuf<MacNode>& out, cudaStream_t st);
void make_batch_geometry(const Partition& P, DBuf<double>& center, DBuf<double>& radius,
                         cudaStream_t st);

// ---------------------------------------------------------------------------
// Interaction lists (engine.py:65-130)
struct Lists {
  int64_t nb = 0;
  int64_t n_groups = 0;
  DBuf<int32_t> a_ptr, d_ptr;   // [nb*G + 1], batch-major then group
  DBuf<int32_t> a_idx, d_idx;   // global cluster ids
  DBuf<int32_t> a_cnt, d_cnt;   // scratch counts
  int64_t n_approx = 0, n_direct = 0;
  DBuf<unsigned long long> pairs;  // [2]: direct, approx
  DBuf<unsigned long long> tot64;  // [2]: list entries (approx, direct) in 64 bits
};

// ---------------------------------------------------------------------------
// Scan utilities
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, DBuf<int32_t>& tmp,
                        cudaStream_t st);

int ceil_div(int64_t a, int64_t b);
// 64-bit sums of two int32 count arrays of n entries (into out[0], out[1],
// zeroed here): the overflow check of the int32 CSR offsets
void sum_counts_i64(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* out,
                    cudaStream_t st);

}  // namespace bltc
