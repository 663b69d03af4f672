// libbltc C ABI (include/bltc.h): contexts, the single-device pipeline that
// replaces treecode_potentials (engine.py:350-372), stage exports for the
// bit-exact checks, and the per-rank entry points of the distributed path
// (decomp.py:483-593).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bltc_internal.cuh"
#include "eval_common.cuh"

namespace bltc {

static thread_local std::string g_err;
std::atomic<long long> g_launch_count{0};
thread_local long long t_launch_count = 0;
void set_error(const std::string& msg) { g_err = msg; }

__global__ void k_moments(const double* sx, const double* sy, const double* sz,
                          const double* sq, const int32_t* list, const int32_t* cstart,
                          const int32_t* cstop, const double* lo, const double* hi,
                          const double* s_nodes, const double* w_nodes, int degree,
                          int mstride, double* rows);
bool launch_moments_k1(const double* sx, const double* sy, const double* sz, const double* sq,
                       const int32_t* list, int64_t n_list, const int32_t* cstart,
                       const int32_t* cstop, const double* lo, const double* hi,
                       const double* s_nodes, const double* w_nodes, int degree, int mstride,
                       double* rows, cudaStream_t st);
bool launch_moments_bw(const double* sx, const double* sy, const double* sz, const double* sq,
                       const int32_t* list, int64_t n_list, const int32_t* cstart,
                       const int32_t* cstop, const double* lo, const double* hi,
                       const double* s_nodes, const double* w_nodes, int degree, int mstride,
                       double* rows, DBuf<int32_t>& cnt, DBuf<int32_t>& off, DBuf<int2>& items,
                       DBuf<int32_t>& scan_tmp, HostScratch& hs, cudaStream_t st,
                       const BwStreams& aux);
__global__ void k_lists(int64_t nb, int G, int g, const double* bcenter, const double* bradius,
                        const int32_t* bstart, const int32_t* bstop, const MacNode* nodes,
                        int32_t cluster_offset, double theta, int64_t per_node, bool fill,
                        int32_t* a_cnt, int32_t* d_cnt, const int32_t* a_ptr,
                        const int32_t* d_ptr, int32_t* a_idx, int32_t* d_idx,
                        unsigned long long* pairs, int32_t* overflow);
__global__ void k_mark_used(int64_t n, const int32_t* idx, int32_t* used);

namespace {

inline int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)(g < 1 ? 1 : g);
}

// Derived cluster geometry (tree.py:46-53, 205-206): center = 0.5 (lo + hi),
// radius = 0.5 sqrt((ex^2 + ey^2) + ez^2), eligible = all extents >= 1e-14.
__global__ void k_mac_nodes(int64_t nn, const double* lo, const double* hi, const int32_t* start,
                            const int32_t* stop, const int32_t* child_start,
                            const int32_t* child_count, MacNode* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  MacNode n;
  double e[3], c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    c[d] = __dmul_rn(0.5, __dadd_rn(lo[3 * i + d], hi[3 * i + d]));
    e[d] = __dsub_rn(hi[3 * i + d], lo[3 * i + d]);
  }
  n.cx = c[0];
  n.cy = c[1];
  n.cz = c[2];
  n.radius = __dmul_rn(
      0.5, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(e[0], e[0]), __dmul_rn(e[1], e[1])),
                                __dmul_rn(e[2], e[2]))));
  n.count = stop[i] - start[i];
  n.child_count = child_count[i];
  n.child_start = child_count[i] ? child_start[i] : -1;
  n.eligible = (e[0] >= kDegenerate && e[1] >= kDegenerate && e[2] >= kDegenerate) ? 1 : 0;
  out[i] = n;
}

__global__ void k_eval_clusters(int64_t nn, const double* lo, const double* hi,
                                const int32_t* start, const int32_t* stop, int32_t offset,
                                EvalCluster* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  EvalCluster c;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    c.lo[d] = lo[3 * i + d];
    c.hi[d] = hi[3 * i + d];
  }
  c.start = start[i] + offset;
  c.stop = stop[i] + offset;
  c.mrow = -1;
  c.pad = 0;
  out[i] = c;
}

__global__ void k_batches(int64_t nb, const int32_t* leaves, const double* lo, const double* hi,
                          const int32_t* start, const int32_t* stop, int32_t* bstart,
                          int32_t* bstop, double* bc, double* br) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int i = leaves[b];
  double e[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    bc[3 * b + d] = __dmul_rn(0.5, __dadd_rn(lo[3 * i + d], hi[3 * i + d]));
    e[d] = __dsub_rn(hi[3 * i + d], lo[3 * i + d]);
  }
  br[b] = __dmul_rn(0.5, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(e[0], e[0]),
                                                        __dmul_rn(e[1], e[1])),
                                              __dmul_rn(e[2], e[2]))));
  bstart[b] = start[i];
  bstop[b] = stop[i];
}

// all == 2 (a rank's publishable rows): every eligible cluster that passes
// the size test and that some batch of the global domain [dlo, dhi] could
// accept geometrically -- a batch ball centred in the domain accepts cluster
// c only if r_B + r_C <= theta |B - C| (engine.py:65-85), so |B - C| >=
// r_C / theta must be reachable inside the domain (dom = nullptr: no filter).
// The domain is a union of n_dom boxes (every batch centre lies in one): the
// cluster keeps its row if r_C / theta is reachable inside any of them.
__global__ void k_flag_moments(int64_t nn, const MacNode* nodes, int64_t per_node, int all,
                               const int32_t* used, int32_t* flag, const double* dom,
                               int64_t n_dom, double theta) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  int f;
  if (all == 1) {
    f = nodes[i].eligible;                                  // compute_all_moments
  } else if (all == 2) {
    const MacNode& m = nodes[i];
    f = m.eligible && per_node < m.count;                   // any possible approx
    if (f && dom) {
      const double c[3] = {m.cx, m.cy, m.cz};
      // generous margins: a cluster on the edge of reach keeps its row
      const double reach = m.radius * (1.0 - 1e-9) / (theta * (1.0 + 1e-9));
      const double reach2 = reach * reach;
      f = 0;
      for (int64_t k = 0; k < n_dom && !f; ++k) {
        const double* b = dom + 6 * k;
        double far2 = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double e = fmax(fabs(b[d] - c[d]), fabs(b[3 + d] - c[d]));
          far2 += e * e;
        }
        f = far2 >= reach2;
      }
    }
  } else {
    f = used[i];
  }
  flag[i] = f;
}

__global__ void k_compact_moments(int64_t nn, const int32_t* flag, const int32_t* pos,
                                  int32_t* list, EvalCluster* ecl) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (flag[i]) {
    list[pos[i]] = (int32_t)i;
    ecl[i].mrow = pos[i];
  }
}

__global__ void k_pack4(int64_t n, const double* x, const double* y, const double* z,
                        const double* q, double4* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double4(x[i], y[i], z[i], q[i]);
}

__global__ void k_unpermute(int64_t n, const double* sorted, const int32_t* perm, double* phi) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) phi[i] = sorted[perm[i]];
}

// Flattened TreeArray record of one cluster (decomp.py:137-189), as doubles
// (all integers < 2^31 are exact): the unit the forest all-gather moves.
constexpr int kRec = 18;
enum RecField {
  R_LO = 0, R_HI = 3, R_CENTER = 6, R_RADIUS = 9, R_COUNT = 10, R_CHILD_START = 11,
  R_CHILD_COUNT = 12, R_ELIGIBLE = 13, R_START = 14, R_STOP = 15, R_MROW = 16
};

__global__ void k_pack_records(int64_t nn, const double* lo, const double* hi,
                               const MacNode* mac, const EvalCluster* ecl, double* rec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  double* r = rec + i * kRec;
  const MacNode m = mac[i];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    r[R_LO + d] = lo[3 * i + d];
    r[R_HI + d] = hi[3 * i + d];
  }
  r[R_CENTER] = m.cx;
  r[R_CENTER + 1] = m.cy;
  r[R_CENTER + 2] = m.cz;
  r[R_RADIUS] = m.radius;
  r[R_COUNT] = m.count;
  r[R_CHILD_START] = m.child_start;
  r[R_CHILD_COUNT] = m.child_count;
  r[R_ELIGIBLE] = m.eligible;
  r[R_START] = ecl[i].start;
  r[R_STOP] = ecl[i].stop;
  r[R_MROW] = ecl[i].mrow;
  r[17] = 0.0;
}

// LET step one: flag every forest cluster some list entry references.
__global__ void k_mark_needs(int64_t n, const int32_t* __restrict__ idx, int bit, int32_t* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicOr(&flags[idx[i]], bit);
}

// One owner's records -> the forest's MacNode / EvalCluster arrays, shifting
// particle ranges and moment rows by the owner's offsets in the forest.
__global__ void k_unpack_records(int64_t nn, const double* rec, int32_t p_off, int32_t row_off,
                                 MacNode* mac, EvalCluster* ecl) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const double* r = rec + i * kRec;
  MacNode m;
  m.cx = r[R_CENTER];
  m.cy = r[R_CENTER + 1];
  m.cz = r[R_CENTER + 2];
  m.radius = r[R_RADIUS];
  m.count = (int32_t)r[R_COUNT];
  m.child_start = (int32_t)r[R_CHILD_START];
  m.child_count = (int32_t)r[R_CHILD_COUNT];
  m.eligible = (int32_t)r[R_ELIGIBLE];
  mac[i] = m;
  EvalCluster c;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    c.lo[d] = r[R_LO + d];
    c.hi[d] = r[R_HI + d];
  }
  c.start = (int32_t)r[R_START] + p_off;
  c.stop = (int32_t)r[R_STOP] + p_off;
  const int32_t mrow = (int32_t)r[R_MROW];
  c.mrow = mrow >= 0 ? mrow + row_off : -1;
  c.pad = 0;
  ecl[i] = c;
}

__global__ void k_widen(int64_t n, const int32_t* a, int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i];
}

}  // namespace
}  // namespace bltc

using namespace bltc;

struct bltc_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  BwStreams bw;   // the bitwise upward pass's auxiliary stream (created on first use)
  // bltc_rank_set_domain: the global domain, to skip moment rows no batch
  // anywhere could read
  // (bltc_rank_set_domain_boxes: a union of boxes, 6 doubles each; empty: unset)
  std::vector<double> domain;
  bool domain_uploaded = false;
  DBuf<double> domain_dev;
  bool timing = true;
  HostScratch hs;
  BuildScratch bs;
  Partition src, tgt_own;
  Partition* tgt = nullptr;
  DBuf<double> in[7];        // H2D staging: tx ty tz sx sy sz q
  DBuf<MacNode> mac;
  DBuf<EvalCluster> ecl;
  DBuf<double> bcenter, bradius;
  DBuf<int32_t> bstart, bstop;
  Lists lists;
  DBuf<int32_t> used, mflag, mpos, mlist;
  DBuf<double> rows;
  int64_t n_moments = 0;
  DBuf<double> s_nodes, w_nodes;
  DBuf<double> out_sorted, far_out, carry, phi_dev;
  DBuf<double4> src4;
  DBuf<int32_t> item_cnt, item_off, counters;
  DBuf<int2> items, items2;
  DBuf<int32_t> pk_pc, pk_poff, pk_wcnt, pk_woff;   // packed FAST items
  DBuf<int4> pk_items;
  PackedOrder pk_order;                              // cost-ordered copies
  DBuf<int32_t> need;   // LET step one flags (bltc_rank_needs)
  DBuf<uint8_t> pk_dmask;
  DBuf<double> partial;
  DBuf<double2> dpartial;
  DBuf<int64_t> didx;
  DBuf<double> dout;
  DBuf<int32_t> flag;
  DBuf<int64_t> widen;
  bltc_params params{};
  bool have_run = false;
  bool lists_staged = false;   // bltc_stage_lists result (exportable lists)
  int64_t launches = 0;
  // distributed: per-rank forest
  bool rank_built = false;
  int64_t rank_n = 0;
  DBuf<EvalCluster> f_ecl;
  DBuf<MacNode> f_mac;
  DBuf<double> f_x, f_y, f_z, f_q, f_rows;
  DBuf<double4> f_src4;
  // STRICT
  DBuf<double> absum;
  StrictScratch strict;
  int64_t n_recomputed = 0;   // -2: count on the device (strict.counters[0]); -1: evaluated as PARITY
};

namespace {

// Validates the parameters and returns them normalised: Yukawa with kappa = 0
// is the Coulomb kernel (exp(-0 r) q / r == q / r bitwise in the reference,
// engine.py:190-191; the FAST / STRICT paths then match Coulomb bitwise too).
bltc_params check_params(const bltc_params* p) {
  if (!p) {
    set_error("params is NULL");
    throw UserError{BLTC_ERR_VALUE};
  }
  if (!(p->theta > 0.0 && p->theta <= 1.0)) {
    set_error("theta must be in (0, 1], got " + std::to_string(p->theta));
    throw UserError{BLTC_ERR_VALUE};
  }
  if (p->degree < 0) {
    set_error("degree must be >= 0");
    throw UserError{BLTC_ERR_VALUE};
  }
  if (p->degree > kMaxDegree) {
    set_error("degree above the supported maximum " + std::to_string(kMaxDegree));
    throw UserError{BLTC_ERR_UNSUPPORTED};
  }
  if (p->leaf_size < 1 || p->batch_size < 1) {
    set_error("leaf_size and batch_size must be >= 1");
    throw UserError{BLTC_ERR_VALUE};
  }
  if (!std::isfinite(p->kappa) || p->kappa < 0.0) {
    set_error("kappa must be finite and >= 0, got " + std::to_string(p->kappa));
    throw UserError{BLTC_ERR_VALUE};
  }
  if (p->kernel_code < 0 || p->kernel_code > 2) {
    set_error("kernel_code must be 0, 1 or 2");
    throw UserError{BLTC_ERR_VALUE};
  }
  if (p->mode != BLTC_MODE_PARITY && p->mode != BLTC_MODE_FAST &&
      p->mode != BLTC_MODE_STRICT) {
    set_error("mode must be BLTC_MODE_PARITY, BLTC_MODE_FAST or BLTC_MODE_STRICT");
    throw UserError{BLTC_ERR_VALUE};
  }
  bltc_params n = *p;
  if (n.kernel_code == 1 && n.kappa == 0.0) n.kernel_code = 0;
  return n;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return BLTC_OK;
  } catch (const UserError& e) {
    return e.code;
  } catch (const CudaFailure&) {
    return BLTC_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(std::string("internal error: ") + e.what());
    return BLTC_ERR_CUDA;
  } catch (...) {
    set_error("unknown internal error");
    return BLTC_ERR_CUDA;
  }
}

struct Timer {
  cudaEvent_t ev[8];
  int n = 0;
  bool on;
  cudaStream_t st;
  Timer(bool enable, cudaStream_t s) : on(enable), st(s) {
    if (on)
      for (auto& e : ev) BLTC_CUDA(cudaEventCreate(&e));
  }
  ~Timer() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
  void mark() {
    if (on) BLTC_CUDA(cudaEventRecord(ev[n++], st));
  }
  double secs(int a, int b) {
    if (!on) return 0.0;
    BLTC_CUDA(cudaEventSynchronize(ev[b]));
    float ms = 0;
    BLTC_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
    return ms * 1e-3;
  }
};

void upload_nodes(bltc_ctx* c, const bltc_params* p, const double* cheb_s) {
  const int m = p->degree + 1;
  std::vector<double> w(m);
  for (int k = 0; k < m; ++k) {   // barycentric_weights (interp.py:59-67)
    double delta = (k == 0 || k == p->degree) ? 0.5 : 1.0;
    w[k] = (k % 2 == 0 ? 1.0 : -1.0) * delta;
  }
  if (p->degree == 0) w[0] = 0.5;
  c->s_nodes.resize(m);
  c->w_nodes.resize(m);
  double* h = (double*)c->hs.get(2 * m * sizeof(double) + 64);
  for (int k = 0; k < m; ++k) {
    h[k] = cheb_s ? cheb_s[k] : 0.0;
    h[m + k] = w[k];
  }
  BLTC_CUDA(cudaMemcpyAsync(c->s_nodes.p, h, m * sizeof(double), cudaMemcpyHostToDevice, c->st));
  BLTC_CUDA(cudaMemcpyAsync(c->w_nodes.p, h + m, m * sizeof(double), cudaMemcpyHostToDevice,
                            c->st));
  BLTC_CUDA(cudaStreamSynchronize(c->st));
}

// Interaction lists of the target batches against one or more source trees
// (groups), CSR batch-major then group.
void build_lists(bltc_ctx* c, const bltc_params* p, int G, const MacNode* const* trees,
                 const int32_t* cluster_offsets) {
  cudaStream_t st = c->st;
  Lists& L = c->lists;
  const int64_t nb = c->bstart.n;
  const int64_t nseg = nb * G;
  const int64_t per_node = (int64_t)(p->degree + 1) * (p->degree + 1) * (p->degree + 1);
  L.nb = nb;
  L.n_groups = G;
  L.a_cnt.resize(nseg + 1);
  L.d_cnt.resize(nseg + 1);
  L.a_ptr.resize(nseg + 1);
  L.d_ptr.resize(nseg + 1);
  L.pairs.resize(2);
  c->flag.resize(1);
  BLTC_CUDA(cudaMemsetAsync(L.pairs.p, 0, 2 * sizeof(unsigned long long), st));
  BLTC_CUDA(cudaMemsetAsync(c->flag.p, 0, sizeof(int32_t), st));
  BLTC_CUDA(cudaMemsetAsync(L.a_cnt.p + nseg, 0, sizeof(int32_t), st));
  BLTC_CUDA(cudaMemsetAsync(L.d_cnt.p + nseg, 0, sizeof(int32_t), st));
  for (int g = 0; g < G; ++g) {
    k_lists<<<grid_for(nb, 64), 64, 0, st>>>(nb, G, g, c->bcenter.p, c->bradius.p, c->bstart.p,
                                             c->bstop.p, trees[g], cluster_offsets[g], p->theta,
                                             per_node, false, L.a_cnt.p, L.d_cnt.p, nullptr,
                                             nullptr, nullptr, nullptr, L.pairs.p, c->flag.p);
    BLTC_LAUNCH_CHECK();
  }
  exclusive_scan_i32(L.a_cnt.p, L.a_ptr.p, nseg + 1, c->bs.scan_tmp, st);
  exclusive_scan_i32(L.d_cnt.p, L.d_ptr.p, nseg + 1, c->bs.scan_tmp, st);
  // the CSR offsets are int32: check the entry totals in 64 bits first
  L.tot64.resize(2);
  sum_counts_i64(L.a_cnt.p, L.d_cnt.p, nseg, L.tot64.p, st);
  int32_t* h = (int32_t*)c->hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, L.a_ptr.p + nseg, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaMemcpyAsync(h + 1, L.d_ptr.p + nseg, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaMemcpyAsync(h + 2, c->flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaMemcpyAsync(h + 4, L.tot64.p, 2 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  if (h[2]) {
    set_error("interaction-list traversal stack overflow (tree too deep)");
    throw UserError{BLTC_ERR_UNSUPPORTED};
  }
  const unsigned long long* t64 = reinterpret_cast<const unsigned long long*>(h + 4);
  if (t64[0] > (unsigned long long)INT32_MAX - 1 || t64[1] > (unsigned long long)INT32_MAX - 1) {
    set_error("interaction lists above 2^31 entries on one device (" + std::to_string(t64[0]) +
              " approximation, " + std::to_string(t64[1]) +
              " direct): split the targets across more ranks");
    throw UserError{BLTC_ERR_UNSUPPORTED};
  }
  L.n_approx = h[0];
  L.n_direct = h[1];
  L.a_idx.resize(L.n_approx + 1);
  L.d_idx.resize(L.n_direct + 1);
  for (int g = 0; g < G; ++g) {
    k_lists<<<grid_for(nb, 64), 64, 0, st>>>(nb, G, g, c->bcenter.p, c->bradius.p, c->bstart.p,
                                             c->bstop.p, trees[g], cluster_offsets[g], p->theta,
                                             per_node, true, nullptr, nullptr, L.a_ptr.p,
                                             L.d_ptr.p, L.a_idx.p, L.d_idx.p, nullptr, c->flag.p);
    BLTC_LAUNCH_CHECK();
  }
}

// Moments of the listed clusters into rows (one row per list entry).  FAST:
// source pieces with fused products, summed piece by piece; PARITY / STRICT:
// bitwise the reference's sums (k_moments_bw; the older one-CTA-per-(cluster,
// k1) and one-CTA-per-cluster kernels remain for degrees 0 and 13-20 and as
// BLTC_MOMENTS_BW=0 / BLTC_PARITY_MOMENTS_OLD=1 measurement switches).
void run_moments(bltc_ctx* c, const bltc_params* p, const double* x, const double* y,
                 const double* z, const double* q, const int32_t* list, int64_t n_list,
                 const int32_t* start, const int32_t* stop, const double* lo, const double* hi,
                 int mstride, double* rows) {
  cudaStream_t st = c->st;
  if (p->mode == BLTC_MODE_FAST) {
    launch_moments_split(x, y, z, q, list, n_list, start, stop, lo, hi, c->s_nodes.p,
                         c->w_nodes.p, p->degree, mstride, rows, c->item_cnt, c->item_off,
                         c->items, c->partial, c->bs.scan_tmp, c->hs, st);
    return;
  }
  if (!c->bw.st) {
    BLTC_CUDA(cudaStreamCreateWithFlags(&c->bw.st, cudaStreamNonBlocking));
    BLTC_CUDA(cudaEventCreateWithFlags(&c->bw.fork, cudaEventDisableTiming));
    BLTC_CUDA(cudaEventCreateWithFlags(&c->bw.join, cudaEventDisableTiming));
  }
  if (launch_moments_bw(x, y, z, q, list, n_list, start, stop, lo, hi, c->s_nodes.p,
                        c->w_nodes.p, p->degree, mstride, rows, c->item_cnt, c->item_off,
                        c->items, c->bs.scan_tmp, c->hs, st, c->bw))
    return;
  const int m = p->degree + 1;
  int threads = ((m * m + 31) / 32) * 32;
  if (threads < 96) threads = 96;
  const char* old_env = std::getenv("BLTC_PARITY_MOMENTS_OLD");
  const bool k1 = !(old_env && std::atoi(old_env) != 0) &&
                  launch_moments_k1(x, y, z, q, list, n_list, start, stop, lo, hi,
                                    c->s_nodes.p, c->w_nodes.p, p->degree, mstride, rows, st);
  if (!k1) {
    k_moments<<<(unsigned)n_list, threads, 0, st>>>(x, y, z, q, list, start, stop, lo, hi,
                                                    c->s_nodes.p, c->w_nodes.p, p->degree,
                                                    mstride, rows);
    BLTC_LAUNCH_CHECK();
  }
}

// Moments of the flagged clusters of one source tree (moments.py:147-150).
// all: 0 = clusters on some approximation list, 1 = every eligible cluster,
// 2 = every cluster the MAC could accept (eligible and (n+1)^3 < N_C).
// The pad double of each moment row (mstride = (n+1)^3 rounded up to even,
// for 16-byte copies) is never written by the upward pass; zero it so the
// evaluation kernels' 16-byte row copies read initialised memory.
void zero_row_pads(double* rows, int64_t n_rows, int degree, int mstride, cudaStream_t st) {
  const int64_t m3 = (int64_t)(degree + 1) * (degree + 1) * (degree + 1);
  if (n_rows <= 0 || mstride == m3) return;
  BLTC_CUDA(cudaMemset2DAsync(rows + m3, mstride * sizeof(double), 0,
                              (mstride - m3) * sizeof(double), n_rows, st));
}

void compute_moments(bltc_ctx* c, const bltc_params* p, const Partition& T, const MacNode* mac,
                     EvalCluster* ecl, int all, DBuf<double>& rows, int64_t cluster_base) {
  cudaStream_t st = c->st;
  const int64_t nn = T.n_nodes;
  const int m = p->degree + 1;
  const int64_t m3 = (int64_t)m * m * m;
  c->used.resize(nn);
  c->mflag.resize(nn + 1);
  c->mpos.resize(nn + 1);
  if (all == 0) {
    BLTC_CUDA(cudaMemsetAsync(c->used.p, 0, nn * sizeof(int32_t), st));
    // approximation entries are global ids; this tree's ids start at cluster_base
    if (c->lists.n_approx > 0) {
      k_mark_used<<<grid_for(c->lists.n_approx, 256), 256, 0, st>>>(
          c->lists.n_approx, c->lists.a_idx.p, c->used.p);
      BLTC_LAUNCH_CHECK();
    }
  }
  (void)cluster_base;
  const double* dom = nullptr;
  const int64_t n_dom = (int64_t)(c->domain.size() / 6);
  if (all == 2 && n_dom > 0) {
    if (!c->domain_uploaded) {
      c->domain_dev.resize(c->domain.size());
      BLTC_CUDA(cudaMemcpyAsync(c->domain_dev.p, c->domain.data(),
                                c->domain.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      c->domain_uploaded = true;
    }
    dom = c->domain_dev.p;
  }
  k_flag_moments<<<grid_for(nn, 256), 256, 0, st>>>(nn, mac, m3, all, c->used.p, c->mflag.p, dom,
                                                    n_dom, p->theta);
  BLTC_LAUNCH_CHECK();
  BLTC_CUDA(cudaMemsetAsync(c->mflag.p + nn, 0, sizeof(int32_t), st));
  exclusive_scan_i32(c->mflag.p, c->mpos.p, nn + 1, c->bs.scan_tmp, st);
  int32_t* h = (int32_t*)c->hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, c->mpos.p + nn, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  c->n_moments = h[0];
  c->mlist.resize(c->n_moments + 1);
  const int mstride = moment_stride(p->degree);
  rows.resize(c->n_moments * mstride + 2);
  zero_row_pads(rows.p, c->n_moments, p->degree, mstride, st);
  k_compact_moments<<<grid_for(nn, 256), 256, 0, st>>>(nn, c->mflag.p, c->mpos.p, c->mlist.p,
                                                       ecl);
  BLTC_LAUNCH_CHECK();
  if (c->n_moments > 0)
    run_moments(c, p, T.x.p, T.y.p, T.z.p, T.q.p, c->mlist.p, c->n_moments, T.start.p, T.stop.p,
                T.lo.p, T.hi.p, mstride, rows.p);
}

void build_batches(bltc_ctx* c, Partition& T) {
  cudaStream_t st = c->st;
  partition_leaves(T, c->bs, st, c->hs);
  const int64_t nb = T.n_leaves;
  c->bstart.resize(nb);
  c->bstop.resize(nb);
  c->bcenter.resize(3 * nb);
  c->bradius.resize(nb);
  k_batches<<<grid_for(nb, 128), 128, 0, st>>>(nb, T.leaves.p, T.lo.p, T.hi.p, T.start.p,
                                               T.stop.p, c->bstart.p, c->bstop.p, c->bcenter.p,
                                               c->bradius.p);
  BLTC_LAUNCH_CHECK();
}

// Potentials of the context's targets (sorted order, c->out_sorted) against
// G source groups.  PARITY: the packed PAR kernels (or k_eval_parity);
// FAST: the packed FAST kernels (or the per-batch ones); STRICT: FAST with
// the near field's |term| sums, then strict_fixup certifies every target or
// recomputes it in the reference's arithmetic (strict.cu).  STRICT without a
// packed instantiation (constant kernel, degrees 0 and 13-20) evaluates as
// PARITY -- bitwise, so trivially within the tolerance.
void evaluate(bltc_ctx* c, const bltc_params* p, int G, const EvalCluster* ecl, const double* sx,
              const double* sy, const double* sz, const double* sq, const double4* src4,
              const double* rows, int64_t n_rows, int64_t n_src, bltc_stats* stats) {
  cudaStream_t st = c->st;
  const Partition& T = *c->tgt;
  EvalArgs a{};
  a.nb = c->bstart.n;
  a.G = G;
  a.bstart = c->bstart.p;
  a.bstop = c->bstop.p;
  a.bcenter = c->bcenter.p;
  a.bradius = c->bradius.p;
  a.tx = T.x.p;
  a.ty = T.y.p;
  a.tz = T.z.p;
  a.a_ptr = c->lists.a_ptr.p;
  a.a_idx = c->lists.a_idx.p;
  a.d_ptr = c->lists.d_ptr.p;
  a.d_idx = c->lists.d_idx.p;
  a.clusters = ecl;
  a.sx = sx;
  a.sy = sy;
  a.sz = sz;
  a.sq = sq;
  a.src4 = src4;
  a.moments = rows;
  a.mstride = moment_stride(p->degree);
  a.s_nodes = c->s_nodes.p;
  a.degree = p->degree;
  a.kappa = p->kappa;
  a.yk = make_yukawa_k(p->kappa);
  c->out_sorted.resize(T.n);
  a.out = c->out_sorted.p;
  a.g_lo = 0;
  a.g_hi = G;
  a.par_first = a.par_last = 1;
  const bool strict = p->mode == BLTC_MODE_STRICT &&
                      packed_supported(p->kernel_code, p->degree);
  // FAST degrees whose per-batch far kernel cannot hold a moment row in
  // shared memory (degree >= 15 without packed kernels) evaluate as PARITY
  const bool fast_ok = p->mode != BLTC_MODE_FAST ||
                       packed_supported(p->kernel_code, p->degree) ||
                       fast_far_fits(p->degree);
  const bool as_parity = p->mode == BLTC_MODE_PARITY ||
                         (p->mode == BLTC_MODE_STRICT && !strict) || !fast_ok;
  c->n_recomputed = as_parity && p->mode == BLTC_MODE_STRICT ? -1 : 0;
  const bool parity_packed = as_parity &&
                             packed_supported(p->kernel_code, p->degree) &&
                             !(std::getenv("BLTC_PARITY_PACKED") &&
                               std::atoi(std::getenv("BLTC_PARITY_PACKED")) == 0);
  if (parity_packed) {
    // bitwise-reference arithmetic on the packed work items: far partials,
    // then the direct sums continuing them (eval_packed.cu, PAR)
    c->far_out.resize(T.n);
    a.far_out = c->far_out.p;
    c->counters.resize(2);
    PackedItems pi;
    build_packed_items(a, c->pk_order, c->pk_pc, c->pk_poff, c->pk_wcnt, c->pk_woff, c->pk_items,
                       c->pk_dmask, c->lists.n_direct, c->bs.scan_tmp, c->hs, st, &pi);
    float far_ms = 0, near_ms = 0;
    if (G > 1) {
      c->carry.resize(T.n);
      a.carry = c->carry.p;
    }
    // one far + near pass per source group, in owner order (decomp.py:437-454)
    for (int g = 0; g < G; ++g) {
      a.g_lo = g;
      a.g_hi = g + 1;
      a.par_first = g == 0;
      a.par_last = g == G - 1;
      float f = 0, n = 0;
      launch_eval_packed(a, p->kernel_code, pi, c->counters.p, st, &f, &n, c->timing, true);
      far_ms += f;
      near_ms += n;
    }
    if (stats) {
      stats->far_s = far_ms * 1e-3;
      stats->near_s = near_ms * 1e-3;
      stats->packed = 1;
    }
  } else if (as_parity) {
    launch_eval_parity(a, p->kernel_code, st);
  } else {
    c->far_out.resize(T.n);
    a.far_out = c->far_out.p;
    float far_ms = 0, near_ms = 0;
    c->counters.resize(2);
    if (packed_supported(p->kernel_code, p->degree)) {
      PackedItems pi;
      build_packed_items(a, c->pk_order, c->pk_pc, c->pk_poff, c->pk_wcnt, c->pk_woff, c->pk_items,
                         c->pk_dmask, c->lists.n_direct, c->bs.scan_tmp, c->hs, st, &pi);
      if (strict || packed_preferred(p->kernel_code, pi.chunk_lane_eff)) {
        if (strict) {
          c->absum.resize(T.n);
          a.absum = c->absum.p;
        }
        launch_eval_packed(a, p->kernel_code, pi, c->counters.p, st, &far_ms, &near_ms,
                           c->timing, false, strict);
        if (strict) {
          cudaEvent_t e0 = nullptr, e1 = nullptr;
          if (c->timing) {
            BLTC_CUDA(cudaEventCreate(&e0));
            BLTC_CUDA(cudaEventCreate(&e1));
            BLTC_CUDA(cudaEventRecord(e0, st));
          }
          strict_fixup(a, p->kernel_code, n_rows, n_src, c->strict, T.n, st);
          c->n_recomputed = -2;   // on the device: read with the stats
          if (c->timing) {
            BLTC_CUDA(cudaEventRecord(e1, st));
            BLTC_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            BLTC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (stats) stats->strict_s = ms * 1e-3;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
          }
        }
        if (stats) {
          stats->far_s = far_ms * 1e-3;
          stats->near_s = near_ms * 1e-3;
          stats->packed = 1;
        }
        return;
      }
    }
    const FastTuning tune = fast_tuning();
    const bool tuned = p->kernel_code == 0;
    const int far_chunk = 32 * (tuned && p->degree == 8 ? tune.far_tpt : 2);
    const int near_chunk = 32 * (tuned ? tune.near_tpt : 2);
    FastItems fi, ni;
    build_fast_items(a, far_chunk, c->item_cnt, c->item_off, c->items, c->bs.scan_tmp, c->hs,
                     st, &fi);
    if (near_chunk == far_chunk) {
      ni = fi;
    } else {
      build_fast_items(a, near_chunk, c->item_cnt, c->item_off, c->items2, c->bs.scan_tmp,
                       c->hs, st, &ni);
    }
    c->counters.resize(2);
    launch_eval_fast(a, p->kernel_code, fi, ni, tune, c->counters.p, st, &far_ms, &near_ms,
                     c->timing);
    if (stats) {
      stats->far_s = far_ms * 1e-3;
      stats->near_s = near_ms * 1e-3;
    }
  }
}

// STRICT: targets recomputed in the reference's arithmetic by the last
// evaluation (-1: evaluated as PARITY; 0 otherwise).  Synchronises.
int64_t read_recomputed(bltc_ctx* c) {
  if (c->n_recomputed != -2) return c->n_recomputed;
  int32_t* h = (int32_t*)c->hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, c->strict.counters.p, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c->st));
  BLTC_CUDA(cudaStreamSynchronize(c->st));
  return h[0];
}

// BLTC_TRACE=1: synchronise and print host wall time per pipeline stage.
struct Trace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t;
  explicit Trace(cudaStream_t s) : on(std::getenv("BLTC_TRACE") != nullptr), st(s) {
    t = std::chrono::steady_clock::now();
  }
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bltc] %-14s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void run_pipeline(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_t,
                  const double* tx, const double* ty, const double* tz, int64_t n_s,
                  const double* sx, const double* sy, const double* sz, const double* q,
                  bool coincident, double* phi_dev, bltc_stats* stats,
                  bool evaluate_phi = true) {
  const bltc_params pn_ = check_params(p);
  p = &pn_;
  if (n_s < 1 || n_t < 1) {
    set_error("cannot partition an empty particle set");
    throw UserError{BLTC_ERR_VALUE};
  }
  if (n_s > (int64_t)INT32_MAX / 2 || n_t > (int64_t)INT32_MAX / 2) {
    set_error("particle count above the supported 2^30 per device");
    throw UserError{BLTC_ERR_UNSUPPORTED};
  }
  cudaStream_t st = c->st;
  c->params = *p;
  c->have_run = false;
  c->lists_staged = false;
  const long long launches0 = t_launch_count;
  Timer tm(c->timing, st);
  upload_nodes(c, p, cheb_s);
  tm.mark();  // 0
  Trace tr(st);
  // ---- setup: source tree, target batches, interaction lists
  build_partition(c->src, c->bs, n_s, sx, sy, sz, q, p->leaf_size, st, c->hs);
  tr("source tree");
  const bool share = coincident && p->batch_size == p->leaf_size;
  if (share) {
    c->tgt = &c->src;   // identical inputs + limits => identical partition (tree.py:225-236)
  } else {
    build_partition(c->tgt_own, c->bs, n_t, coincident ? sx : tx, coincident ? sy : ty,
                    coincident ? sz : tz, nullptr, p->batch_size, st, c->hs);
    c->tgt = &c->tgt_own;
  }
  tr("target tree");
  build_batches(c, *c->tgt);
  tr("batches");
  const int64_t nn = c->src.n_nodes;
  c->mac.resize(nn);
  c->ecl.resize(nn);
  k_mac_nodes<<<grid_for(nn, 128), 128, 0, st>>>(nn, c->src.lo.p, c->src.hi.p, c->src.start.p,
                                                 c->src.stop.p, c->src.child_start.p,
                                                 c->src.child_count.p, c->mac.p);
  BLTC_LAUNCH_CHECK();
  k_eval_clusters<<<grid_for(nn, 128), 128, 0, st>>>(nn, c->src.lo.p, c->src.hi.p,
                                                     c->src.start.p, c->src.stop.p, 0, c->ecl.p);
  BLTC_LAUNCH_CHECK();
  const MacNode* trees[1] = {c->mac.p};
  const int32_t offs[1] = {0};
  build_lists(c, p, 1, trees, offs);
  tr("lists");
  tm.mark();  // 1
  // ---- precompute: moments
  compute_moments(c, p, c->src, c->mac.p, c->ecl.p, p->all_moments ? 1 : 0, c->rows, 0);
  tr("moments");
  tm.mark();  // 2
  // ---- compute: evaluation + un-permute (skipped by bltc_build)
  if (evaluate_phi) {
  {   // packed (x, y, z, q) records: FAST and the packed PARITY kernels
    c->src4.resize(n_s);
    k_pack4<<<grid_for(n_s, 256), 256, 0, st>>>(n_s, c->src.x.p, c->src.y.p, c->src.z.p,
                                                c->src.q.p, c->src4.p);
    BLTC_LAUNCH_CHECK();
  }
  evaluate(c, p, 1, c->ecl.p, c->src.x.p, c->src.y.p, c->src.z.p, c->src.q.p, c->src4.p,
           c->rows.p, c->n_moments, n_s, stats);
  k_unpermute<<<grid_for(n_t, 256), 256, 0, st>>>(n_t, c->out_sorted.p, c->tgt->perm.p, phi_dev);
  BLTC_LAUNCH_CHECK();
  tr("evaluate");
  }
  tm.mark();  // 3
  if (stats) {
    unsigned long long* h = (unsigned long long*)c->hs.get(64);
    BLTC_CUDA(cudaMemcpyAsync(h, c->lists.pairs.p, 2 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
    BLTC_CUDA(cudaStreamSynchronize(st));
    stats->n_clusters = nn;
    stats->n_batches = c->bstart.n;
    stats->direct_pairs = (int64_t)h[0];
    stats->approx_pairs = (int64_t)h[1];
    stats->setup_s = tm.secs(0, 1);
    stats->precompute_s = tm.secs(1, 2);
    stats->compute_s = tm.secs(2, 3);
    stats->total_s = tm.secs(0, 3);
    stats->n_moments = c->n_moments;
    stats->kernel_launches = t_launch_count - launches0;
    stats->tree_depth = c->src.depth;
    stats->batch_depth = c->tgt->depth;
    stats->n_recomputed = read_recomputed(c);
  } else {
    BLTC_CUDA(cudaStreamSynchronize(st));
  }
  c->have_run = true;
}

void require_run(bltc_ctx* c) {
  if (!c || !c->have_run) {
    set_error("no completed run on this context");
    throw UserError{BLTC_ERR_STATE};
  }
}

template <typename T>
void d2h(T* host, const T* dev, int64_t n, cudaStream_t st) {
  if (host && n > 0) BLTC_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}

void d2h_widen(bltc_ctx* c, int64_t* host, const int32_t* dev, int64_t n) {
  if (!host || n <= 0) return;
  c->widen.resize(n);
  k_widen<<<grid_for(n, 256), 256, 0, c->st>>>(n, dev, c->widen.p);
  BLTC_LAUNCH_CHECK();
  d2h(host, c->widen.p, n, c->st);
  BLTC_CUDA(cudaStreamSynchronize(c->st));
}


// ---- host-structure stage calls: upload helpers ---------------------------
template <typename T>
void h2d(DBuf<T>& dst, const T* src, int64_t n, cudaStream_t st) {
  dst.resize(n > 0 ? n : 1);
  if (n > 0) BLTC_CUDA(cudaMemcpyAsync(dst.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

// int64 host indices -> int32 device buffer (values must fit, checked)
void h2d_narrow(DBuf<int32_t>& dst, const int64_t* src, int64_t n, cudaStream_t st,
                const char* what) {
  std::vector<int32_t> tmp(n > 0 ? n : 1);
  for (int64_t i = 0; i < n; ++i) {
    if (src[i] < INT32_MIN || src[i] > INT32_MAX) {
      set_error(std::string(what) + " value out of the supported int32 range");
      throw UserError{BLTC_ERR_UNSUPPORTED};
    }
    tmp[i] = (int32_t)src[i];
  }
  dst.resize(n > 0 ? n : 1);
  if (n > 0) {
    BLTC_CUDA(cudaMemcpyAsync(dst.p, tmp.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice,
                              st));
    BLTC_CUDA(cudaStreamSynchronize(st));   // tmp goes out of scope
  }
}

void require_ptr(const void* ptr, const char* what) {
  if (!ptr) {
    set_error(std::string(what) + " is NULL");
    throw UserError{BLTC_ERR_VALUE};
  }
}

// Upload a source tree given as BFS arrays (tree.py:198-217 / bltc_export_tree)
// into c->src and derive the MAC / evaluation records.
void upload_tree(bltc_ctx* c, int64_t nc, const int64_t* start, const int64_t* stop,
                 const double* lo, const double* hi, const int64_t* child_start,
                 const int64_t* child_count) {
  cudaStream_t st = c->st;
  Partition& S = c->src;
  h2d_narrow(S.start, start, nc, st, "cluster start");
  h2d_narrow(S.stop, stop, nc, st, "cluster stop");
  h2d_narrow(S.child_start, child_start, nc, st, "child_start");
  h2d_narrow(S.child_count, child_count, nc, st, "child_count");
  h2d(S.lo, lo, 3 * nc, st);
  h2d(S.hi, hi, 3 * nc, st);
  S.n_nodes = nc;
  c->mac.resize(nc);
  c->ecl.resize(nc);
  k_mac_nodes<<<grid_for(nc, 128), 128, 0, st>>>(nc, S.lo.p, S.hi.p, S.start.p, S.stop.p,
                                                 S.child_start.p, S.child_count.p, c->mac.p);
  BLTC_LAUNCH_CHECK();
  k_eval_clusters<<<grid_for(nc, 128), 128, 0, st>>>(nc, S.lo.p, S.hi.p, S.start.p, S.stop.p, 0,
                                                     c->ecl.p);
  BLTC_LAUNCH_CHECK();
}

void upload_batches(bltc_ctx* c, int64_t nb, const int64_t* bstart, const int64_t* bstop,
                    const double* bcenter, const double* bradius) {
  h2d_narrow(c->bstart, bstart, nb, c->st, "batch start");
  h2d_narrow(c->bstop, bstop, nb, c->st, "batch stop");
  c->bstart.n = c->bstop.n = nb;
  h2d(c->bcenter, bcenter, 3 * nb, c->st);
  h2d(c->bradius, bradius, nb, c->st);
}

}  // namespace

extern "C" {


const char* bltc_last_error(void) { return g_err.c_str(); }
const char* bltc_version(void) { return "libbltc 0.1 (sm_100a)"; }

int bltc_create(int device, void* stream, bltc_ctx** out) {
  return guarded([&] {
    if (!out) {
      set_error("out is NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    bltc_ctx* c = new bltc_ctx();
    if (device < 0) BLTC_CUDA(cudaGetDevice(&device));
    c->device = device;
    BLTC_CUDA(cudaSetDevice(device));
    if (stream) {
      c->st = (cudaStream_t)stream;
    } else {
      BLTC_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    *out = c;
  });
}

int bltc_destroy(bltc_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    Partition* ps[2] = {&c->src, &c->tgt_own};
    for (Partition* P : ps) {
      P->x.release(); P->y.release(); P->z.release(); P->q.release(); P->order.release();
      P->perm.release(); P->start.release(); P->stop.release(); P->child_start.release();
      P->child_count.release(); P->level.release(); P->lo.release(); P->hi.release();
      P->leaves.release();
    }
    BuildScratch& S = c->bs;
    S.x1.release(); S.y1.release(); S.z1.release(); S.q1.release(); S.o1.release();
    S.node_of0.release(); S.node_of1.release(); S.code.release(); S.tile_cnt.release();
    S.node_base.release(); S.node_off.release(); S.node_child.release(); S.node_nchild.release();
    S.node_split.release(); S.node_mid.release(); S.box_u.release(); S.scan_tmp.release();
    S.counter.release();
    for (auto& b : c->in) b.release();
    c->mac.release(); c->ecl.release(); c->bcenter.release(); c->bradius.release();
    c->bstart.release(); c->bstop.release();
    Lists& L = c->lists;
    L.a_ptr.release(); L.d_ptr.release(); L.a_idx.release(); L.d_idx.release();
    L.a_cnt.release(); L.d_cnt.release(); L.pairs.release();
    c->used.release(); c->mflag.release(); c->mpos.release(); c->mlist.release();
    c->rows.release(); c->s_nodes.release(); c->w_nodes.release(); c->out_sorted.release();
    c->far_out.release(); c->carry.release(); c->phi_dev.release(); c->src4.release(); c->flag.release();
    c->widen.release(); c->item_cnt.release(); c->item_off.release(); c->counters.release();
    c->items.release(); c->items2.release();
    c->pk_pc.release(); c->pk_poff.release(); c->pk_wcnt.release(); c->pk_woff.release();
    c->pk_items.release(); c->pk_dmask.release();
    c->pk_order.far.release(); c->pk_order.near.release(); c->pk_order.cost.release();
    c->pk_order.cost_sorted.release(); c->pk_order.tmp.release(); c->need.release(); c->partial.release(); c->dpartial.release();
    c->didx.release(); c->dout.release(); c->f_ecl.release(); c->f_mac.release(); c->f_x.release();
    c->f_y.release(); c->f_z.release(); c->f_q.release(); c->f_rows.release();
    c->f_src4.release();
    c->hs.release();
    c->domain_dev.release();
    if (c->bw.st) {
      cudaStreamDestroy(c->bw.st);
      cudaEventDestroy(c->bw.fork);
      cudaEventDestroy(c->bw.join);
    }
    if (c->own_stream) cudaStreamDestroy(c->st);
    delete c;
  });
}

int bltc_set_timing(bltc_ctx* c, int enable) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    c->timing = enable != 0;
  });
}

int bltc_treecode_device(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_t,
                         const double* tx, const double* ty, const double* tz, int64_t n_s,
                         const double* sx, const double* sy, const double* sz, const double* q,
                         int32_t coincident, double* phi_out, bltc_stats* stats) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    BLTC_CUDA(cudaSetDevice(c->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    run_pipeline(c, p, cheb_s, n_t, tx, ty, tz, n_s, sx, sy, sz, q, coincident != 0, phi_out,
                 stats);
  });
}

int bltc_build(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_t,
               const double* tx, const double* ty, const double* tz, int64_t n_s,
               const double* sx, const double* sy, const double* sz, const double* q,
               int32_t coincident, bltc_stats* stats) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    BLTC_CUDA(cudaSetDevice(c->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    if (n_s < 1 || n_t < 1) {
      set_error("cannot partition an empty particle set");
      throw UserError{BLTC_ERR_VALUE};
    }
    require_ptr(sx, "sx");
    require_ptr(sy, "sy");
    require_ptr(sz, "sz");
    require_ptr(q, "q");
    if (!coincident) {
      require_ptr(tx, "tx");
      require_ptr(ty, "ty");
      require_ptr(tz, "tz");
    }
    cudaStream_t st = c->st;
    const double* hs_[7] = {tx, ty, tz, sx, sy, sz, q};
    const int64_t ns_[7] = {n_t, n_t, n_t, n_s, n_s, n_s, n_s};
    for (int k = 0; k < 7; ++k) {
      if (coincident && k < 3) continue;
      c->in[k].resize(ns_[k]);
      BLTC_CUDA(cudaMemcpyAsync(c->in[k].p, hs_[k], ns_[k] * sizeof(double),
                                cudaMemcpyHostToDevice, st));
    }
    const bool co = coincident != 0;
    run_pipeline(c, p, cheb_s, n_t, co ? c->in[3].p : c->in[0].p, co ? c->in[4].p : c->in[1].p,
                 co ? c->in[5].p : c->in[2].p, n_s, c->in[3].p, c->in[4].p, c->in[5].p,
                 c->in[6].p, co, nullptr, stats, false);
  });
}

int bltc_treecode(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_t,
                  const double* tx, const double* ty, const double* tz, int64_t n_s,
                  const double* sx, const double* sy, const double* sz, const double* q,
                  int32_t coincident, double* phi_out, bltc_stats* stats) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    BLTC_CUDA(cudaSetDevice(c->device));
    if (stats) std::memset(stats, 0, sizeof(*stats));
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    if (n_s < 1 || n_t < 1) {
      set_error("cannot partition an empty particle set");
      throw UserError{BLTC_ERR_VALUE};
    }
    cudaStream_t st = c->st;
    cudaEvent_t e0, e1, e2, e3;
    BLTC_CUDA(cudaEventCreate(&e0));
    BLTC_CUDA(cudaEventCreate(&e1));
    BLTC_CUDA(cudaEventCreate(&e2));
    BLTC_CUDA(cudaEventCreate(&e3));
    BLTC_CUDA(cudaEventRecord(e0, st));
    const double* hs_[7] = {tx, ty, tz, sx, sy, sz, q};
    const int64_t ns_[7] = {n_t, n_t, n_t, n_s, n_s, n_s, n_s};
    for (int k = 0; k < 7; ++k) {
      if (coincident && k < 3) continue;
      c->in[k].resize(ns_[k]);
      BLTC_CUDA(cudaMemcpyAsync(c->in[k].p, hs_[k], ns_[k] * sizeof(double),
                                cudaMemcpyHostToDevice, st));
    }
    BLTC_CUDA(cudaEventRecord(e1, st));
    c->phi_dev.resize(n_t);
    const bool co = coincident != 0;
    run_pipeline(c, p, cheb_s, n_t, co ? c->in[3].p : c->in[0].p, co ? c->in[4].p : c->in[1].p,
                 co ? c->in[5].p : c->in[2].p, n_s, c->in[3].p, c->in[4].p, c->in[5].p,
                 c->in[6].p, co, c->phi_dev.p, stats);
    BLTC_CUDA(cudaEventRecord(e2, st));
    BLTC_CUDA(cudaMemcpyAsync(phi_out, c->phi_dev.p, n_t * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
    BLTC_CUDA(cudaEventRecord(e3, st));
    BLTC_CUDA(cudaEventSynchronize(e3));
    float a = 0, b = 0;
    BLTC_CUDA(cudaEventElapsedTime(&a, e0, e1));
    BLTC_CUDA(cudaEventElapsedTime(&b, e2, e3));
    if (stats) {
      stats->h2d_s = a * 1e-3;
      stats->d2h_s = b * 1e-3;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
  });
}

int bltc_get_sizes(bltc_ctx* c, bltc_sizes* out) {
  return guarded([&] {
    require_run(c);
    out->n_sources = c->src.n;
    out->n_targets = c->tgt->n;
    out->n_clusters = c->src.n_nodes;
    out->n_batches = c->bstart.n;
    out->n_approx = c->lists.n_approx;
    out->n_direct = c->lists.n_direct;
    out->n_moments = c->n_moments;
    out->degree = c->params.degree;
    out->tree_depth = c->src.depth;
    out->batch_depth = c->tgt->depth;
    out->n_groups = (int32_t)c->lists.n_groups;
  });
}

int bltc_export_tree(bltc_ctx* c, int which, int64_t* n_nodes_out, int64_t* perm, int64_t* start,
                     int64_t* stop, double* lo, double* hi, int64_t* child_start,
                     int64_t* child_count, int32_t* level) {
  return guarded([&] {
    require_run(c);
    BLTC_CUDA(cudaSetDevice(c->device));
    const Partition& P = which == 0 ? c->src : *c->tgt;
    if (n_nodes_out) *n_nodes_out = P.n_nodes;
    d2h_widen(c, perm, P.perm.p, P.n);
    d2h_widen(c, start, P.start.p, P.n_nodes);
    d2h_widen(c, stop, P.stop.p, P.n_nodes);
    d2h_widen(c, child_start, P.child_start.p, P.n_nodes);
    d2h_widen(c, child_count, P.child_count.p, P.n_nodes);
    d2h(lo, P.lo.p, 3 * P.n_nodes, c->st);
    d2h(hi, P.hi.p, 3 * P.n_nodes, c->st);
    d2h(level, P.level.p, P.n_nodes, c->st);
    BLTC_CUDA(cudaStreamSynchronize(c->st));
  });
}

int bltc_export_batches(bltc_ctx* c, int64_t* start, int64_t* stop, double* center,
                        double* radius) {
  return guarded([&] {
    require_run(c);
    BLTC_CUDA(cudaSetDevice(c->device));
    const int64_t nb = c->bstart.n;
    d2h_widen(c, start, c->bstart.p, nb);
    d2h_widen(c, stop, c->bstop.p, nb);
    d2h(center, c->bcenter.p, 3 * nb, c->st);
    d2h(radius, c->bradius.p, nb, c->st);
    BLTC_CUDA(cudaStreamSynchronize(c->st));
  });
}

int bltc_export_lists(bltc_ctx* c, int64_t* a_ptr, int64_t* a_idx, int64_t* d_ptr,
                      int64_t* d_idx) {
  return guarded([&] {
    if (!(c && c->lists_staged)) require_run(c);
    BLTC_CUDA(cudaSetDevice(c->device));
    const Lists& L = c->lists;
    const int64_t nseg = L.nb * L.n_groups;
    d2h_widen(c, a_ptr, L.a_ptr.p, nseg + 1);
    d2h_widen(c, d_ptr, L.d_ptr.p, nseg + 1);
    d2h_widen(c, a_idx, L.a_idx.p, L.n_approx);
    d2h_widen(c, d_idx, L.d_idx.p, L.n_direct);
  });
}

int bltc_export_moments(bltc_ctx* c, int64_t* cluster_ids, double* rows) {
  return guarded([&] {
    require_run(c);
    BLTC_CUDA(cudaSetDevice(c->device));
    const int m = c->params.degree + 1;
    const size_t m3 = (size_t)m * m * m;
    d2h_widen(c, cluster_ids, c->mlist.p, c->n_moments);
    if (rows && c->n_moments > 0)
      BLTC_CUDA(cudaMemcpy2DAsync(rows, m3 * sizeof(double), c->rows.p,
                                  moment_stride(c->params.degree) * sizeof(double),
                                  m3 * sizeof(double), c->n_moments, cudaMemcpyDeviceToHost,
                                  c->st));
    BLTC_CUDA(cudaStreamSynchronize(c->st));
  });
}

int bltc_strict_keep_bounds(bltc_ctx* c, int32_t enable) {
  return guarded([&] {
    if (!c) {
      set_error("ctx is NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    c->strict.want_bounds = enable != 0;
  });
}

int bltc_export_strict_bounds(bltc_ctx* c, double* bounds_out, double* kc_out) {
  return guarded([&] {
    require_run(c);
    if (kc_out) *kc_out = c->strict.kc_used;
    if (c->n_recomputed != -2 || !c->strict.want_bounds || c->rank_built) {
      set_error("no STRICT single-device run with bltc_strict_keep_bounds enabled");
      throw UserError{BLTC_ERR_STATE};
    }
    BLTC_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->tgt->n;
    if (bounds_out && n > 0) {
      c->phi_dev.resize(n);
      k_unpermute<<<grid_for(n, 256), 256, 0, c->st>>>(n, c->strict.bounds.p, c->tgt->perm.p,
                                                       c->phi_dev.p);
      BLTC_LAUNCH_CHECK();
      BLTC_CUDA(cudaMemcpyAsync(bounds_out, c->phi_dev.p, n * sizeof(double),
                                cudaMemcpyDeviceToHost, c->st));
    }
    BLTC_CUDA(cudaStreamSynchronize(c->st));
  });
}

int bltc_direct_sum(bltc_ctx* c, int32_t kernel_code, double kappa, int32_t mode,
                    int64_t n_idx, const int64_t* idx, int64_t n_t, const double* tx,
                    const double* ty, const double* tz, int64_t n_s, const double* sx,
                    const double* sy, const double* sz, const double* q, double* out) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    if (kernel_code < 0 || kernel_code > 2 || !std::isfinite(kappa) || kappa < 0.0 ||
        n_t < 1 || n_s < 1 || n_idx < 0) {
      set_error("invalid direct-sum arguments");
      throw UserError{BLTC_ERR_VALUE};
    }
    BLTC_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    const double* hs_[7] = {tx, ty, tz, sx, sy, sz, q};
    const int64_t ns_[7] = {n_t, n_t, n_t, n_s, n_s, n_s, n_s};
    for (int k = 0; k < 7; ++k) {
      c->in[k].resize(ns_[k]);
      BLTC_CUDA(cudaMemcpyAsync(c->in[k].p, hs_[k], ns_[k] * sizeof(double),
                                cudaMemcpyHostToDevice, st));
    }
    const int64_t m = idx ? n_idx : n_t;
    c->didx.resize(m);
    if (idx) {
      BLTC_CUDA(cudaMemcpyAsync(c->didx.p, idx, m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    } else {
      std::vector<int64_t> all(m);
      for (int64_t i = 0; i < m; ++i) all[i] = i;
      BLTC_CUDA(cudaMemcpyAsync(c->didx.p, all.data(), m * sizeof(int64_t),
                                cudaMemcpyHostToDevice, st));
      BLTC_CUDA(cudaStreamSynchronize(st));
    }
    c->dout.resize(m);
    direct_sum_device(kernel_code, kappa, mode, m, c->didx.p, c->in[0].p, c->in[1].p,
                      c->in[2].p, n_s, c->in[3].p, c->in[4].p, c->in[5].p, c->in[6].p,
                      c->dout.p, c->src4, c->dpartial, st);
    BLTC_CUDA(cudaMemcpyAsync(out, c->dout.p, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    BLTC_CUDA(cudaStreamSynchronize(st));
  });
}

int bltc_rank_build(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n,
                    const double* x, const double* y, const double* z, const double* q,
                    int32_t device_ptrs) {
  return guarded([&] {
    if (!c) throw UserError{BLTC_ERR_VALUE};
    BLTC_CUDA(cudaSetDevice(c->device));
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    if (n < 1) {
      set_error("cannot partition an empty particle set");
      throw UserError{BLTC_ERR_VALUE};
    }
    cudaStream_t st = c->st;
    c->params = *p;
    c->have_run = false;
    c->rank_built = false;
    const double* dx = x;
    const double* dy = y;
    const double* dz = z;
    const double* dq = q;
    if (!device_ptrs) {
      const double* hs_[4] = {x, y, z, q};
      for (int k = 0; k < 4; ++k) {
        c->in[3 + k].resize(n);
        BLTC_CUDA(cudaMemcpyAsync(c->in[3 + k].p, hs_[k], n * sizeof(double),
                                  cudaMemcpyHostToDevice, st));
      }
      dx = c->in[3].p;
      dy = c->in[4].p;
      dz = c->in[5].p;
      dq = c->in[6].p;
    }
    Timer tm(c->timing, st);
    upload_nodes(c, p, cheb_s);
    tm.mark();
    // local tree + local batches (decomp.py:507-520)
    build_partition(c->src, c->bs, n, dx, dy, dz, dq, p->leaf_size, st, c->hs);
    if (p->batch_size == p->leaf_size) {
      c->tgt = &c->src;
    } else {
      build_partition(c->tgt_own, c->bs, n, dx, dy, dz, nullptr, p->batch_size, st, c->hs);
      c->tgt = &c->tgt_own;
    }
    build_batches(c, *c->tgt);
    const int64_t nn = c->src.n_nodes;
    c->mac.resize(nn);
    c->ecl.resize(nn);
    k_mac_nodes<<<grid_for(nn, 128), 128, 0, st>>>(nn, c->src.lo.p, c->src.hi.p, c->src.start.p,
                                                   c->src.stop.p, c->src.child_start.p,
                                                   c->src.child_count.p, c->mac.p);
    BLTC_LAUNCH_CHECK();
    k_eval_clusters<<<grid_for(nn, 128), 128, 0, st>>>(nn, c->src.lo.p, c->src.hi.p,
                                                       c->src.start.p, c->src.stop.p, 0, c->ecl.p);
    BLTC_LAUNCH_CHECK();
    tm.mark();
    // moments of every cluster another rank's MAC could accept (decomp.py:526-533;
    // the reference publishes all eligible rows, only these can ever be read)
    compute_moments(c, p, c->src, c->mac.p, c->ecl.p, 2, c->rows, 0);
    tm.mark();
    BLTC_CUDA(cudaStreamSynchronize(st));
    c->rank_n = n;
    c->rank_built = true;
  });
}

int bltc_rank_set_domain_boxes(bltc_ctx* c, int64_t n_boxes, const double* boxes) {
  return guarded([&] {
    if (!c || n_boxes < 0 || (n_boxes > 0 && !boxes)) throw UserError{BLTC_ERR_VALUE};
    for (int64_t k = 0; k < n_boxes; ++k)
      for (int d = 0; d < 3; ++d) {
        const double lo = boxes[6 * k + d], hi = boxes[6 * k + 3 + d];
        if (!std::isfinite(lo) || !std::isfinite(hi) || lo > hi) {
          set_error("domain boxes must be finite with lo <= hi");
          throw UserError{BLTC_ERR_VALUE};
        }
      }
    c->domain.assign(boxes, boxes + 6 * n_boxes);
    c->domain_uploaded = false;
  });
}

int bltc_rank_set_domain(bltc_ctx* c, const double* lo, const double* hi) {
  if (!lo || !hi) return bltc_rank_set_domain_boxes(c, 0, nullptr);
  const double box[6] = {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]};
  return bltc_rank_set_domain_boxes(c, 1, box);
}

int bltc_domain_cells(int64_t n, const double* x, const double* y, const double* z, int32_t grid,
                      double* boxes, int64_t* n_boxes) {
  return guarded([&] {
    if (n < 1 || !x || !y || !z || grid < 1 || grid > 64 || !boxes || !n_boxes)
      throw UserError{BLTC_ERR_VALUE};
    const double* P[3] = {x, y, z};
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = hi[d] = P[d][0];
      for (int64_t i = 1; i < n; ++i) {
        lo[d] = std::min(lo[d], P[d][i]);
        hi[d] = std::max(hi[d], P[d][i]);
      }
      if (!std::isfinite(lo[d]) || !std::isfinite(hi[d])) {
        set_error("coordinates must be finite");
        throw UserError{BLTC_ERR_VALUE};
      }
    }
    const int64_t G = grid, nc = G * G * G;
    std::vector<double> cb(6 * nc);
    std::vector<char> occ(nc, 0);
    for (int64_t i = 0; i < n; ++i) {
      int64_t cell = 0;
      for (int d = 0; d < 3; ++d) {
        const double w = hi[d] - lo[d];
        int64_t k = w > 0 ? (int64_t)((P[d][i] - lo[d]) / w * G) : 0;
        k = std::min<int64_t>(std::max<int64_t>(k, 0), G - 1);
        cell = cell * G + k;
      }
      double* b = &cb[6 * cell];
      if (!occ[cell]) {
        occ[cell] = 1;
        for (int d = 0; d < 3; ++d) b[d] = b[3 + d] = P[d][i];
      } else {
        for (int d = 0; d < 3; ++d) {
          b[d] = std::min(b[d], P[d][i]);
          b[3 + d] = std::max(b[3 + d], P[d][i]);
        }
      }
    }
    int64_t m = 0;
    for (int64_t cell = 0; cell < nc; ++cell)
      if (occ[cell]) {
        std::copy(&cb[6 * cell], &cb[6 * cell] + 6, boxes + 6 * m);
        ++m;
      }
    *n_boxes = m;
  });
}

int bltc_rank_publish_sizes(bltc_ctx* c, bltc_publish_sizes* out) {
  return guarded([&] {
    if (!c || !c->rank_built) {
      set_error("bltc_rank_build has not run on this context");
      throw UserError{BLTC_ERR_STATE};
    }
    out->n_clusters = c->src.n_nodes;
    out->n_particles = c->rank_n;
    out->n_moment_rows = c->n_moments;
    out->record_doubles = kRec;
  });
}

int bltc_rank_publish(bltc_ctx* c, double* records, double* particles, double* moments) {
  return guarded([&] {
    if (!c || !c->rank_built) {
      set_error("bltc_rank_build has not run on this context");
      throw UserError{BLTC_ERR_STATE};
    }
    BLTC_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    const int64_t nn = c->src.n_nodes, n = c->rank_n;
    k_pack_records<<<grid_for(nn, 128), 128, 0, st>>>(nn, c->src.lo.p, c->src.hi.p, c->mac.p,
                                                      c->ecl.p, records);
    BLTC_LAUNCH_CHECK();
    const double* src[4] = {c->src.x.p, c->src.y.p, c->src.z.p, c->src.q.p};
    for (int k = 0; k < 4; ++k)
      BLTC_CUDA(cudaMemcpyAsync(particles + k * n, src[k], n * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    const int mstride = moment_stride(c->params.degree);
    if (c->n_moments > 0)
      BLTC_CUDA(cudaMemcpyAsync(moments, c->rows.p, c->n_moments * mstride * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    BLTC_CUDA(cudaStreamSynchronize(st));
  });
}

int bltc_rank_needs(bltc_ctx* c, const bltc_params* p, int32_t ranks, int32_t my_rank,
                    const int64_t* n_clusters, const double* const* records, int32_t* flags_out) {
  return guarded([&] {
    if (!c || !c->rank_built) {
      set_error("bltc_rank_build has not run on this context");
      throw UserError{BLTC_ERR_STATE};
    }
    BLTC_CUDA(cudaSetDevice(c->device));
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    if (ranks < 1 || my_rank < 0 || my_rank >= ranks) {
      set_error("invalid ranks / my_rank");
      throw UserError{BLTC_ERR_VALUE};
    }
    if (p->degree != c->params.degree || p->leaf_size != c->params.leaf_size ||
        p->batch_size != c->params.batch_size) {
      set_error("list parameters differ from those of bltc_rank_build");
      throw UserError{BLTC_ERR_VALUE};
    }
    cudaStream_t st = c->st;
    std::vector<int> owners;
    owners.push_back(my_rank);
    for (int o = 0; o < ranks; ++o)
      if (o != my_rank) owners.push_back(o);
    const int G = ranks;
    std::vector<int32_t> cl_off(G), rank_off(ranks);
    int64_t C = 0;
    for (int g = 0; g < G; ++g) {
      cl_off[g] = (int32_t)C;
      C += n_clusters[owners[g]];
    }
    int64_t R0 = 0;
    for (int o = 0; o < ranks; ++o) {
      rank_off[o] = (int32_t)R0;
      R0 += n_clusters[o];
    }
    c->f_mac.resize(C);
    c->f_ecl.resize(C);
    std::vector<const MacNode*> trees(G);
    for (int g = 0; g < G; ++g) {
      const int64_t nc = n_clusters[owners[g]];
      k_unpack_records<<<grid_for(nc, 128), 128, 0, st>>>(nc, records[owners[g]], 0, 0,
                                                          c->f_mac.p + cl_off[g],
                                                          c->f_ecl.p + cl_off[g]);
      BLTC_LAUNCH_CHECK();
      trees[g] = c->f_mac.p + cl_off[g];
    }
    build_lists(c, p, G, trees.data(), cl_off.data());
    c->need.resize(C + 1);
    BLTC_CUDA(cudaMemsetAsync(c->need.p, 0, (C + 1) * sizeof(int32_t), st));
    const Lists& L = c->lists;
    if (L.n_approx > 0) {
      k_mark_needs<<<grid_for(L.n_approx, 256), 256, 0, st>>>(L.n_approx, L.a_idx.p, 1,
                                                               c->need.p);
      BLTC_LAUNCH_CHECK();
    }
    if (L.n_direct > 0) {
      k_mark_needs<<<grid_for(L.n_direct, 256), 256, 0, st>>>(L.n_direct, L.d_idx.p, 2,
                                                               c->need.p);
      BLTC_LAUNCH_CHECK();
    }
    for (int g = 0; g < G; ++g) {
      const int o = owners[g];
      if (n_clusters[o] > 0)
        BLTC_CUDA(cudaMemcpyAsync(flags_out + rank_off[o], c->need.p + cl_off[g],
                                  n_clusters[o] * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                  st));
    }
    BLTC_CUDA(cudaStreamSynchronize(st));
  });
}

int bltc_rank_evaluate(bltc_ctx* c, const bltc_params* p, int32_t ranks, int32_t my_rank,
                       const int64_t* n_clusters, const int64_t* n_particles,
                       const int64_t* n_moment_rows, const double* const* records,
                       const double* const* particles, const double* const* moments,
                       double* phi_out, int32_t device_ptrs, bltc_stats* stats) {
  return guarded([&] {
    if (!c || !c->rank_built) {
      set_error("bltc_rank_build has not run on this context");
      throw UserError{BLTC_ERR_STATE};
    }
    BLTC_CUDA(cudaSetDevice(c->device));
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    if (ranks < 1 || my_rank < 0 || my_rank >= ranks) {
      set_error("invalid ranks / my_rank");
      throw UserError{BLTC_ERR_VALUE};
    }
    if (p->degree != c->params.degree || p->leaf_size != c->params.leaf_size ||
        p->batch_size != c->params.batch_size) {
      set_error("evaluation parameters differ from those of bltc_rank_build");
      throw UserError{BLTC_ERR_VALUE};
    }
    if (stats) std::memset(stats, 0, sizeof(*stats));
    cudaStream_t st = c->st;
    const long long launches0 = t_launch_count;
    Timer tm(c->timing, st);
    tm.mark();
    // owner order of _eval_rank (decomp.py:437-454): local first, then the
    // remote owners ascending
    std::vector<int> owners;
    owners.push_back(my_rank);
    for (int o = 0; o < ranks; ++o)
      if (o != my_rank) owners.push_back(o);
    const int G = ranks;
    const int mstride = moment_stride(p->degree);
    std::vector<int32_t> cl_off(G), p_off(G), row_off(G);
    int64_t C = 0, P = 0, RW = 0;
    for (int g = 0; g < G; ++g) {
      const int o = owners[g];
      cl_off[g] = (int32_t)C;
      p_off[g] = (int32_t)P;
      row_off[g] = (int32_t)RW;
      C += n_clusters[o];
      P += n_particles[o];
      RW += n_moment_rows[o];
    }
    if (P > (int64_t)INT32_MAX / 2) {
      set_error("forest above 2^30 particles per device");
      throw UserError{BLTC_ERR_UNSUPPORTED};
    }
    c->f_mac.resize(C);
    c->f_ecl.resize(C);
    c->f_x.resize(P);
    c->f_y.resize(P);
    c->f_z.resize(P);
    c->f_q.resize(P);
    c->f_rows.resize(RW * mstride + 2);
    std::vector<const MacNode*> trees(G);
    for (int g = 0; g < G; ++g) {
      const int o = owners[g];
      const int64_t nc = n_clusters[o], np = n_particles[o];
      k_unpack_records<<<grid_for(nc, 128), 128, 0, st>>>(nc, records[o], p_off[g], row_off[g],
                                                          c->f_mac.p + cl_off[g],
                                                          c->f_ecl.p + cl_off[g]);
      BLTC_LAUNCH_CHECK();
      double* dst[4] = {c->f_x.p, c->f_y.p, c->f_z.p, c->f_q.p};
      for (int k = 0; k < 4; ++k)
        BLTC_CUDA(cudaMemcpyAsync(dst[k] + p_off[g], particles[o] + k * np, np * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
      if (n_moment_rows[o] > 0)
        BLTC_CUDA(cudaMemcpyAsync(c->f_rows.p + (size_t)row_off[g] * mstride, moments[o],
                                  n_moment_rows[o] * mstride * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
      trees[g] = c->f_mac.p + cl_off[g];
    }
    c->params = *p;
    build_lists(c, p, G, trees.data(), cl_off.data());
    tm.mark();
    {   // packed (x, y, z, q) records: FAST and the packed PARITY kernels
      c->f_src4.resize(P);
      k_pack4<<<grid_for(P, 256), 256, 0, st>>>(P, c->f_x.p, c->f_y.p, c->f_z.p, c->f_q.p,
                                                c->f_src4.p);
      BLTC_LAUNCH_CHECK();
    }
    evaluate(c, p, G, c->f_ecl.p, c->f_x.p, c->f_y.p, c->f_z.p, c->f_q.p, c->f_src4.p,
             c->f_rows.p, RW, P, stats);
    const int64_t n = c->rank_n;
    c->phi_dev.resize(n);
    k_unpermute<<<grid_for(n, 256), 256, 0, st>>>(n, c->out_sorted.p, c->tgt->perm.p,
                                                  device_ptrs ? phi_out : c->phi_dev.p);
    BLTC_LAUNCH_CHECK();
    if (!device_ptrs)
      BLTC_CUDA(cudaMemcpyAsync(phi_out, c->phi_dev.p, n * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
    tm.mark();
    unsigned long long* h = (unsigned long long*)c->hs.get(64);
    BLTC_CUDA(cudaMemcpyAsync(h, c->lists.pairs.p, 2 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
    BLTC_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      stats->n_clusters = c->src.n_nodes;
      stats->n_batches = c->bstart.n;
      stats->direct_pairs = (int64_t)h[0];
      stats->approx_pairs = (int64_t)h[1];
      stats->setup_s = tm.secs(0, 1);
      stats->compute_s = tm.secs(1, 2);
      stats->total_s = tm.secs(0, 2);
      stats->n_moments = c->n_moments;
      stats->kernel_launches = t_launch_count - launches0;
      stats->tree_depth = c->src.depth;
      stats->batch_depth = c->tgt->depth;
      stats->n_recomputed = read_recomputed(c);
    }
    c->have_run = true;
  });
}

// ---- Stage calls with host-provided upstream structures -------------------

int bltc_stage_lists(bltc_ctx* c, const bltc_params* p, int64_t n_batches,
                     const int64_t* batch_start, const int64_t* batch_stop,
                     const double* batch_center, const double* batch_radius,
                     int64_t n_clusters, const int64_t* start, const int64_t* stop,
                     const double* lo, const double* hi, const int64_t* child_start,
                     const int64_t* child_count, int64_t* n_approx, int64_t* n_direct) {
  return guarded([&] {
    if (!c) {
      set_error("ctx is NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    BLTC_CUDA(cudaSetDevice(c->device));
    if (n_batches < 1 || n_clusters < 1) {
      set_error("need at least one batch and one cluster");
      throw UserError{BLTC_ERR_VALUE};
    }
    for (const void* q : {(const void*)batch_start, (const void*)batch_stop,
                          (const void*)batch_center, (const void*)batch_radius,
                          (const void*)start, (const void*)stop, (const void*)lo,
                          (const void*)hi, (const void*)child_start,
                          (const void*)child_count})
      require_ptr(q, "stage input");
    c->have_run = false;
    c->params = *p;
    upload_batches(c, n_batches, batch_start, batch_stop, batch_center, batch_radius);
    upload_tree(c, n_clusters, start, stop, lo, hi, child_start, child_count);
    const MacNode* trees[1] = {c->mac.p};
    const int32_t offs[1] = {0};
    build_lists(c, p, 1, trees, offs);
    BLTC_CUDA(cudaStreamSynchronize(c->st));
    if (n_approx) *n_approx = c->lists.n_approx;
    if (n_direct) *n_direct = c->lists.n_direct;
    c->lists_staged = true;
  });
}

int bltc_stage_moments(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_s,
                       const double* sx, const double* sy, const double* sz, const double* q,
                       int64_t n_clusters, const int64_t* start, const int64_t* stop,
                       const double* lo, const double* hi, int64_t n_list,
                       const int64_t* cluster_ids, double* rows_out) {
  return guarded([&] {
    if (!c) {
      set_error("ctx is NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    BLTC_CUDA(cudaSetDevice(c->device));
    if (n_s < 1 || n_clusters < 1) {
      set_error("need at least one source and one cluster");
      throw UserError{BLTC_ERR_VALUE};
    }
    for (const void* ptr : {(const void*)sx, (const void*)sy, (const void*)sz, (const void*)q,
                            (const void*)start, (const void*)stop, (const void*)lo,
                            (const void*)hi})
      require_ptr(ptr, "stage input");
    if (n_list > 0) {
      require_ptr(cluster_ids, "cluster_ids");
      require_ptr(rows_out, "rows_out");
    }
    c->have_run = false;
    c->params = *p;
    cudaStream_t st = c->st;
    upload_nodes(c, p, cheb_s);
    Partition& S = c->src;
    h2d(S.x, sx, n_s, st);
    h2d(S.y, sy, n_s, st);
    h2d(S.z, sz, n_s, st);
    h2d(S.q, q, n_s, st);
    S.n = n_s;
    h2d_narrow(S.start, start, n_clusters, st, "cluster start");
    h2d_narrow(S.stop, stop, n_clusters, st, "cluster stop");
    h2d(S.lo, lo, 3 * n_clusters, st);
    h2d(S.hi, hi, 3 * n_clusters, st);
    for (int64_t i = 0; i < n_list; ++i)
      if (cluster_ids[i] < 0 || cluster_ids[i] >= n_clusters) {
        set_error("cluster id out of range");
        throw UserError{BLTC_ERR_VALUE};
      }
    h2d_narrow(c->mlist, cluster_ids, n_list, st, "cluster id");
    if (n_list == 0) return;
    const int m = p->degree + 1;
    const int64_t m3 = (int64_t)m * m * m;
    const int mstride = moment_stride(p->degree);
    c->rows.resize(n_list * mstride + 2);
    zero_row_pads(c->rows.p, n_list, p->degree, mstride, st);
    run_moments(c, p, S.x.p, S.y.p, S.z.p, S.q.p, c->mlist.p, n_list, S.start.p, S.stop.p,
                S.lo.p, S.hi.p, mstride, c->rows.p);
    BLTC_CUDA(cudaMemcpy2DAsync(rows_out, m3 * sizeof(double), c->rows.p,
                                mstride * sizeof(double), m3 * sizeof(double), n_list,
                                cudaMemcpyDeviceToHost, st));
    BLTC_CUDA(cudaStreamSynchronize(st));
  });
}

int bltc_stage_potentials(bltc_ctx* c, const bltc_params* p, const double* cheb_s, int64_t n_t,
                          const double* tx, const double* ty, const double* tz,
                          int64_t n_batches, const int64_t* batch_start,
                          const int64_t* batch_stop, const double* batch_center,
                          const double* batch_radius, int64_t n_s, const double* sx,
                          const double* sy, const double* sz, const double* q,
                          int64_t n_clusters, const int64_t* start, const int64_t* stop,
                          const double* lo, const double* hi, const int64_t* a_ptr,
                          const int64_t* a_idx, const int64_t* d_ptr, const int64_t* d_idx,
                          const int64_t* moment_row, int64_t n_rows, const double* rows,
                          const int64_t* perm, double* phi_out, bltc_stats* stats) {
  return guarded([&] {
    if (!c) {
      set_error("ctx is NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    const bltc_params pn_ = check_params(p);
    p = &pn_;
    BLTC_CUDA(cudaSetDevice(c->device));
    if (n_t < 1 || n_s < 1 || n_batches < 1 || n_clusters < 1) {
      set_error("need targets, sources, batches and clusters");
      throw UserError{BLTC_ERR_VALUE};
    }
    for (const void* ptr : {(const void*)tx, (const void*)ty, (const void*)tz,
                            (const void*)batch_start, (const void*)batch_stop,
                            (const void*)batch_center, (const void*)batch_radius,
                            (const void*)sx, (const void*)sy, (const void*)sz, (const void*)q,
                            (const void*)start, (const void*)stop, (const void*)lo,
                            (const void*)hi, (const void*)a_ptr, (const void*)d_ptr,
                            (const void*)moment_row, (const void*)phi_out})
      require_ptr(ptr, "stage input");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    c->have_run = false;
    c->params = *p;
    cudaStream_t st = c->st;
    const long long launches0 = t_launch_count;
    Timer tm(c->timing, st);
    upload_nodes(c, p, cheb_s);
    tm.mark();
    const int m = p->degree + 1;
    const int64_t m3 = (int64_t)m * m * m;
    const int mstride = moment_stride(p->degree);
    // batches must tile valid target ranges, the CSR offsets be monotone and
    // perm index the targets (bad caller structures must not reach the device)
    for (int64_t b = 0; b < n_batches; ++b) {
      if (batch_start[b] < 0 || batch_stop[b] > n_t || batch_start[b] > batch_stop[b]) {
        set_error("batch target range out of bounds");
        throw UserError{BLTC_ERR_VALUE};
      }
      if (a_ptr[b] < 0 || a_ptr[b + 1] < a_ptr[b] || d_ptr[b] < 0 || d_ptr[b + 1] < d_ptr[b]) {
        set_error("list offsets (a_ptr / d_ptr) must be non-negative and non-decreasing");
        throw UserError{BLTC_ERR_VALUE};
      }
    }
    if (perm)
      for (int64_t i = 0; i < n_t; ++i)
        if (perm[i] < 0 || perm[i] >= n_t) {
          set_error("perm entry out of range");
          throw UserError{BLTC_ERR_VALUE};
        }
    // targets (batch order) and batches
    Partition& T = c->tgt_own;
    h2d(T.x, tx, n_t, st);
    h2d(T.y, ty, n_t, st);
    h2d(T.z, tz, n_t, st);
    T.n = n_t;
    c->tgt = &T;
    upload_batches(c, n_batches, batch_start, batch_stop, batch_center, batch_radius);
    // sources (cluster order) and clusters
    Partition& S = c->src;
    h2d(S.x, sx, n_s, st);
    h2d(S.y, sy, n_s, st);
    h2d(S.z, sz, n_s, st);
    h2d(S.q, q, n_s, st);
    S.n = n_s;
    S.n_nodes = n_clusters;
    std::vector<EvalCluster> ecl(n_clusters);
    for (int64_t i = 0; i < n_clusters; ++i) {
      EvalCluster& e = ecl[i];
      for (int d = 0; d < 3; ++d) {
        e.lo[d] = lo[3 * i + d];
        e.hi[d] = hi[3 * i + d];
      }
      if (start[i] < 0 || stop[i] > n_s || start[i] > stop[i]) {
        set_error("cluster particle range out of bounds");
        throw UserError{BLTC_ERR_VALUE};
      }
      e.start = (int32_t)start[i];
      e.stop = (int32_t)stop[i];
      if (moment_row[i] >= n_rows) {
        set_error("moment row out of range");
        throw UserError{BLTC_ERR_VALUE};
      }
      e.mrow = (int32_t)moment_row[i];
      e.pad = 0;
    }
    c->ecl.resize(n_clusters);
    BLTC_CUDA(cudaMemcpyAsync(c->ecl.p, ecl.data(), n_clusters * sizeof(EvalCluster),
                              cudaMemcpyHostToDevice, st));
    // lists (single source group) and pair counts (engine.py:133-143)
    Lists& L = c->lists;
    const int64_t na = a_ptr[n_batches], nd = d_ptr[n_batches];
    if ((na > 0 && !a_idx) || (nd > 0 && !d_idx)) {
      set_error("list entries are NULL");
      throw UserError{BLTC_ERR_VALUE};
    }
    unsigned long long approx_pairs = 0, direct_pairs = 0;
    for (int64_t b = 0; b < n_batches; ++b) {
      const int64_t nt_b = batch_stop[b] - batch_start[b];
      for (int64_t e = a_ptr[b]; e < a_ptr[b + 1]; ++e) {
        if (a_idx[e] < 0 || a_idx[e] >= n_clusters || moment_row[a_idx[e]] < 0) {
          set_error("approximation entry without a moment row");
          throw UserError{BLTC_ERR_VALUE};
        }
        approx_pairs += (unsigned long long)(nt_b * m3);
      }
      for (int64_t e = d_ptr[b]; e < d_ptr[b + 1]; ++e) {
        if (d_idx[e] < 0 || d_idx[e] >= n_clusters) {
          set_error("direct entry out of range");
          throw UserError{BLTC_ERR_VALUE};
        }
        direct_pairs += (unsigned long long)(nt_b * (stop[d_idx[e]] - start[d_idx[e]]));
      }
    }
    h2d_narrow(L.a_ptr, a_ptr, n_batches + 1, st, "a_ptr");
    h2d_narrow(L.d_ptr, d_ptr, n_batches + 1, st, "d_ptr");
    h2d_narrow(L.a_idx, a_idx, na, st, "a_idx");
    h2d_narrow(L.d_idx, d_idx, nd, st, "d_idx");
    L.nb = n_batches;
    L.n_groups = 1;
    L.n_approx = na;
    L.n_direct = nd;
    // moments, rows padded to the 16-byte stride
    c->rows.resize(n_rows * mstride + 2);
    if (n_rows > 0) {
      require_ptr(rows, "rows");
      BLTC_CUDA(cudaMemcpy2DAsync(c->rows.p, mstride * sizeof(double), rows,
                                  m3 * sizeof(double), m3 * sizeof(double), n_rows,
                                  cudaMemcpyHostToDevice, st));
    }
    {   // packed (x, y, z, q) records: FAST and the packed PARITY kernels
      c->src4.resize(n_s);
      k_pack4<<<grid_for(n_s, 256), 256, 0, st>>>(n_s, S.x.p, S.y.p, S.z.p, S.q.p, c->src4.p);
      BLTC_LAUNCH_CHECK();
    }
    tm.mark();
    evaluate(c, p, 1, c->ecl.p, S.x.p, S.y.p, S.z.p, S.q.p, c->src4.p, c->rows.p, n_rows, n_s,
             stats);
    c->phi_dev.resize(n_t);
    if (perm) {   // (out + carry)[perm] of compute_potentials (engine.py:335)
      h2d_narrow(T.perm, perm, n_t, st, "perm");
      k_unpermute<<<grid_for(n_t, 256), 256, 0, st>>>(n_t, c->out_sorted.p, T.perm.p,
                                                      c->phi_dev.p);
      BLTC_LAUNCH_CHECK();
      BLTC_CUDA(cudaMemcpyAsync(phi_out, c->phi_dev.p, n_t * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
    } else {
      BLTC_CUDA(cudaMemcpyAsync(phi_out, c->out_sorted.p, n_t * sizeof(double),
                                cudaMemcpyDeviceToHost, st));
    }
    tm.mark();
    BLTC_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      stats->n_clusters = n_clusters;
      stats->n_batches = n_batches;
      stats->direct_pairs = (int64_t)direct_pairs;
      stats->approx_pairs = (int64_t)approx_pairs;
      stats->compute_s = tm.secs(1, 2);
      stats->total_s = tm.secs(0, 2);
      stats->n_moments = n_rows;
      stats->kernel_launches = t_launch_count - launches0;
      stats->n_recomputed = read_recomputed(c);
    }
  });
}

}  // extern "C"
