// FAST-mode evaluation with packed work items (the default FAST path).
//
// Target batches are octree leaves with at most N_B targets but usually far
// fewer (C4, N_B = 500: median 105).  Splitting each batch into 64-target
// chunks leaves lanes idle on every ragged tail (~10% of the lanes at
// N_B = 500, ~18% at N_B = 250).  Here the batches' targets, each batch
// padded to an even count, form one stream of target slots; a work item is
// a 64-slot window of that stream (two targets per lane) and may span up to
// kGMax consecutive batches ("segments").  Each lane walks its own batch's
// interaction list; in step e every segment processes entry e of its own
// list, so lanes stay converged, and a lane whose list has ended simply
// discards its per-cluster partial.  Consecutive batches are octree
// neighbours with similar lists, so little work is lost to ragged list
// lengths (C4: 98.6% of the far-field lane work is useful at N_B = 500,
// 97.6% at N_B = 250, against 90.5% / 81.8% for per-batch chunks).
//
//   far field  (_approx_tile, engine.py:216-252): per segment, the
//     cluster's proxy points and its moment row (k1 slabs of (n+1)^2
//     values, double-buffered with cp.async) are staged in the warp's shared
//     memory; every lane reads its own segment's copy (broadcast loads).
//   near field (_direct_tile, engine.py:151-213): per segment, the sources of
//     its direct list form one stream (cluster after cluster, list order),
//     staged kNearCh packed (x, y, z, q) records at a time (double-
//     buffered); exhausted streams are padded with zero-charge records far
//     away, which add exactly 0.
// FAST arithmetic: rsqrt seed + cubic correction, the charge / moment as the
// operand a lane's two targets share (FORM 2), 7 / 12 FP64 slots per far /
// near pair; Yukawa with the table-driven exp (eval_common.cuh).  PAR: the
// same items and staging with the reference's arithmetic and order, bitwise
// (one source group; the distributed forest uses eval_parity.cu).
// Measured choices: kGMax = 4, two targets per lane, 8 warps x
// 2 CTAs per SM (register bound), k2 unrolled by 3, dy^2 in shared memory.
#include <cub/device/device_radix_sort.cuh>

#include "bltc_internal.cuh"
#include "eval_common.cuh"
#include "exp2w_table.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace bltc {

namespace {
constexpr int kWarps = 8;     // warps per CTA
#ifndef BLTC_GMAX
#define BLTC_GMAX 4
#endif
constexpr int kGMax = BLTC_GMAX;   // batches (segments) per work item
constexpr int kSlots = 64;    // target slots per item: 2 per lane
constexpr int kNearCh = 32;   // near field default: sources per staged chunk and segment

__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double xy = __dmul_rn(x, y);
  const double e = fma(-xy, y, 1.0);
  const double c = fma(0.375, e, 0.5);
  const double ye = __dmul_rn(y, e);
  return fma(ye, c, y);
}

// q / sqrt(d2) accumulated into acc (eval_fast.cu: one 3-register DFMA).
// FORM 0: acc += (q y0) p.  FORM 2: acc += q (y0 p) -- the charge / moment
// is the operand shared by a lane's two targets, so the second accumulating
// DFMA can take it from the operand reuse cache (two register reads).
template <int FORM>
__device__ __forceinline__ double coulomb_acc(double acc, double q, double d2) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d2));
  const double e = fma(-__dmul_rn(d2, y0), y0, 1.0);
  const double c = fma(0.375, e, 0.5);
  const double p = fma(e, c, 1.0);
  if (FORM == 2) return fma(q, __dmul_rn(y0, p), acc);
  const double qy = __dmul_rn(q, y0);
  return fma(qy, p, acc);
}

template <int KIND, int FORM = 0>
__device__ __forceinline__ double pair_acc(double acc, double q, double d2, const YukawaK& yk) {
  if (KIND == 0) return coulomb_acc<FORM>(acc, q, d2);
  const double y = rsqrt_fast(d2);
  const double r = __dmul_rn(d2, y);
  const double ex = exp_neg_kr(r, yk);
  if (FORM == 2) return fma(q, __dmul_rn(ex, y), acc);
  return fma(__dmul_rn(q, ex), y, acc);
}

// The FAST kernel factor f with term = q f (FORM 2): Coulomb y0 p, Yukawa
// exp(-kappa r) y -- the same roundings as pair_acc<KIND, 2>.  STRICT's near
// field accumulates both q f and |q| f.
template <int KIND>
__device__ __forceinline__ double pair_factor(double d2, const YukawaK& yk) {
  if (KIND == 0) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d2));
    const double e = fma(-__dmul_rn(d2, y0), y0, 1.0);
    const double c = fma(0.375, e, 0.5);
    const double p = fma(e, c, 1.0);
    return __dmul_rn(y0, p);
  }
  const double y = rsqrt_fast(d2);
  const double r = __dmul_rn(d2, y);
  return __dmul_rn(exp_neg_kr(r, yk), y);
}

// PARITY: the reference tiles' term, IEEE sqrt / division, no contraction
// (engine.py:183-191, 240-244).
template <int KIND>
__device__ __forceinline__ double parity_term(double q, double d2, double kappa) {
  if (KIND == 0) return __ddiv_rn(q, __dsqrt_rn(d2));
  const double r = __dsqrt_rn(d2);
  return __ddiv_rn(__dmul_rn(libm_exp(__dmul_rn(-kappa, r)), q), r);
}

// Coulomb PARITY term q / sqrt(d2) on the intrinsics' fast paths (bitwise
// __ddiv_rn(q, __dsqrt_rn(d2)) when ok; 0 / s is exactly q for q = +-0).
__device__ __forceinline__ double coulomb_parity_fp(double q, double d2, bool& ok) {
  bool ok1, ok2;
  const double sq = sqrt_rn_fastpath(d2, ok1);
  const double t = div_rn_fastpath(q, sq, ok2);
  const bool zero = q == 0.0;
  ok = ok1 && (ok2 || zero);
  return zero ? q : t;
}

__device__ __forceinline__ void neumaier(double& acc, double& comp, double t) {
  const double s = __dadd_rn(acc, t);
  const bool big = fabs(acc) >= fabs(t);
  const double hi = big ? acc : t, lo = big ? t : acc;
  comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(hi, s), lo));
  acc = s;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Bulk (TMA-engine) copies global -> shared with mbarrier completion
// (cp.async.bulk, SASS UBLKCP): one instruction moves a whole contiguous run.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int next_item(int* counter) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, it, 0);
}

// First index j in [0, n] with a[j] > v (a non-decreasing).
__device__ __forceinline__ int64_t upper_bound(const int32_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] > v) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Work items.  pc[b] = batch size rounded up to even; poff = exclusive scan
// (slot offset of each batch, poff[nb] = total slots S).  Window w covers
// slots [64 w, min(64 w + 64, S)); a window overlapping more than kGMax
// batches is split into several items.  Item = {slot_begin, slot_end,
// first batch, segments}.
// Also accumulates the lane slots the per-batch chunking of eval_fast.cu
// would use (64-target chunks, a tail of <= 32 on half a warp), to choose
// between the two decompositions.
__global__ void k_pad_counts(int64_t nb, const int32_t* bstart, const int32_t* bstop,
                             int32_t* pc, unsigned long long* acc2) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long slots = 0, targets = 0;
  if (b < nb) {
    const int n = bstop[b] - bstart[b];
    pc[b] = n + (n & 1);
    const int r = n % kSlots;
    slots = (unsigned long long)(n - r) + (r > 32 ? kSlots : (r > 0 ? 32 : 0));
    targets = (unsigned long long)n;
  } else if (b == nb) {
    pc[b] = 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    slots += __shfl_xor_sync(0xffffffffu, slots, o);
    targets += __shfl_xor_sync(0xffffffffu, targets, o);
  }
  if ((threadIdx.x & 31) == 0 && slots) {
    atomicAdd(&acc2[0], slots);
    atomicAdd(&acc2[1], targets);
  }
}

__device__ __forceinline__ void window_batches(int64_t nb, const int32_t* poff, int64_t w,
                                               int64_t* s0, int64_t* s1, int64_t* bf,
                                               int64_t* bl) {
  const int64_t S = poff[nb];
  *s0 = w * kSlots;
  *s1 = min(*s0 + kSlots, S);
  *bf = upper_bound(poff, nb, *s0) - 1;
  *bl = upper_bound(poff, nb, *s1 - 1) - 1;
}

__global__ void k_window_counts(int64_t nb, const int32_t* poff, int64_t nw, int32_t* cnt) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w < nw) {
    int64_t s0, s1, bf, bl;
    window_batches(nb, poff, w, &s0, &s1, &bf, &bl);
    cnt[w] = (int32_t)((bl - bf + kGMax) / kGMax);
  } else if (w == nw) {
    cnt[w] = 0;
  }
}

__global__ void k_window_fill(int64_t nb, const int32_t* poff, int64_t nw, const int32_t* ioff,
                              int4* items) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nw) return;
  int64_t s0, s1, bf, bl;
  window_batches(nb, poff, w, &s0, &s1, &bf, &bl);
  int32_t o = ioff[w];
  for (int64_t ba = bf; ba <= bl; ba += kGMax) {
    const int64_t be = min(ba + kGMax, bl + 1);   // exclusive
    const int64_t sb = max(s0, (int64_t)poff[ba]);
    const int64_t se = min(s1, (int64_t)poff[be]);
    items[o++] = make_int4((int)sb, (int)se, (int)ba, (int)(be - ba));
  }
}

// Per direct-list entry: can a pair of (batch, cluster) be singular?  The
// singular-pair test (d^2 < 1e-28, engine.py:175) can only fire if the
// batch ball comes within ~1e-14 of the cluster box.
// Also, per batch (bys): can the Yukawa near field use the shifted-exp table
// with s = 0 -- every pair of the batch's direct list within c r + 2 <= 2048
// (r <= |batch center - cluster center| + batch radius + half diagonal)?
__global__ void k_direct_mask(int64_t nb, int G, const int32_t* d_ptr, const int32_t* d_idx,
                              const EvalCluster* clusters, const double* bcenter,
                              const double* bradius, uint8_t* mask, double c2, uint8_t* bys) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const double* bc = bcenter + 3 * b;
  const double br = bradius[b];
  const double scale = fmax(fmax(fabs(bc[0]), fabs(bc[1])), fabs(bc[2])) + br;
  bool ys = true;
  for (int e = d_ptr[b * G]; e < d_ptr[(b + 1) * G]; ++e) {
    const EvalCluster& c = clusters[d_idx[e]];
    double g2 = 0.0, cd2 = 0.0, hd2 = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double lo = c.lo[d] - bc[d], hi = bc[d] - c.hi[d];
      const double g = fmax(fmax(lo, hi), 0.0);
      g2 = fma(g, g, g2);
      const double cc = 0.5 * (c.lo[d] + c.hi[d]) - bc[d], ex = 0.5 * (c.hi[d] - c.lo[d]);
      cd2 = fma(cc, cc, cd2);
      hd2 = fma(ex, ex, hd2);
    }
    ys &= c2 * (sqrt(cd2) + br + sqrt(hd2)) * (1.0 + 1e-12) + 2.0 <= (double)kExp2WK;
    mask[e] = (sqrt(g2) - br) <= 1e-12 * (1.0 + scale) ? 1 : 0;
#ifdef BLTC_DEBUG_NOMASK
    mask[e] = 0;   // timing experiment only: wrong results for singular pairs
#endif
  }
  bys[b] = ys ? 1 : 0;
}

// Lane layout of one item: slots slot_begin + 2 lane, +1.
struct LaneTargets {
  int g;          // segment of this lane
  int i0, i1;     // target indices (i1 == i0 when the second slot is padding)
  bool v0, v1;    // slot holds a real target
};

__device__ __forceinline__ LaneTargets lane_targets(const int4 it, const EvalArgs& a,
                                                    const int32_t* poff, int lane) {
  LaneTargets L;
  int s = it.x + 2 * lane;
  const bool on = s < it.y;
  if (!on) s = it.x;
  L.g = 0;
#pragma unroll
  for (int k = 1; k < kGMax; ++k)
    if (k < it.w && s >= poff[it.z + k]) L.g = k;
  const int b = it.z + L.g;
  L.i0 = a.bstart[b] + (s - poff[b]);
  const int stop = a.bstop[b];
  L.v0 = on;
  L.v1 = on && (L.i0 + 1 < stop);
  L.i1 = L.v1 ? L.i0 + 1 : L.i0;
  return L;
}

// ---------------------------------------------------------------------------
// Far field.  Shared memory per warp: a header with each segment's list
// range and current moment row (kept out of registers: the pair loop needs
// them for its ILP), then per segment the proxy points [3][M] and two k1
// slabs of M*M moments; segment regions are offset by one double so that
// lanes of different segments read different banks.
template <int M>
struct FarSmem {
  static constexpr int kHdr = 2 * kGMax;                     // doubles
  static constexpr int kPts = 3 * M;
  static constexpr int kSlab = M * M;
  static constexpr int kSeg = kPts + 2 * kSlab + 1;          // doubles per segment
  static constexpr int kWarp = kHdr + kGMax * kSeg + 1;      // doubles per warp
  static constexpr int kDy = 2 * M * 32;                     // DY: dy^2 [M][2][32 lanes]
};

struct FarHdr {
  int e0[kGMax];
  int len[kGMax];
  const double* row[kGMax];   // current moment row (nullptr: segment idle)
};
static_assert(sizeof(FarHdr) <= 2 * kGMax * sizeof(double) + kGMax * sizeof(double),
              "far header");

template <int M>
__device__ __forceinline__ void far_stage_slab(double* wsm, const FarHdr* H, int k1, int lane) {
  using SM = FarSmem<M>;
#pragma unroll
  for (int k = 0; k < kGMax; ++k) {
    const double* row = H->row[k];
    if (row != nullptr) {
      double* slab = wsm + SM::kHdr + k * SM::kSeg + SM::kPts + (k1 & 1) * SM::kSlab;
      const double* src = row + (size_t)k1 * SM::kSlab;
      for (int i = lane; i < SM::kSlab; i += 32) cp_async8(slab + i, src + i);
    }
  }
  cp_async_commit();
}

// PAR: bitwise the reference's _approx_tile (per cluster a plain sum in k1,
// k2, k3 order, then out += acc per cluster in list order): d2 unfused,
// IEEE sqrt / division.
// DY: dy^2 per (target, k2) computed once per cluster into lane-private
// shared-memory slots, so a row costs one DADD per target (dx^2 + dy^2)
// instead of a DSUB and a DFMA.
// FAST Yukawa far field with a shifted exponential (YS): per (target,
// cluster) s = rint(c r_ref), r_ref = |target - box center|, c = kappa 2048 /
// ln2, so that for every proxy point exp(-kappa r) = 2^(-s/2048) 2^(w/2048),
// w = s - c r, |w| <= c hd + 1 (hd: the box's half diagonal).  With S = magic
// + s, z = RN(S - c r) is magic + k (k = rint(w): the low word), S - z = s - k
// exactly and f = w - k = fma(r, -c, S - z): the table T[k] = 2^(k/2048)
// (kExp2W, |k| <= 2048, staged in shared memory) times a degree-3 Taylor
// polynomial of 2^(f/2048) (truncation 3.4e-17) -- no exponent assembly and
// no clamp in the pair loop (16 FP64 slots per pair instead of 17, and ~5
// fewer integer instructions); the 2^(-s/2048) factor is applied once per
// (target, cluster).  Clusters with c hd + 2 > 2048, or targets with
// c r_ref >= 2^30, take the generic exp_neg_kr path for that step.
struct YsState {
  double S;    // magic + s
  double E;    // 2^(-s/2048)
  int si;      // s (< 2^30)
};

// S - z = s - k is formed in the integer pipe and converted (I2F), not by a
// DADD on the FP64 pipe: one FP64 slot less per pair.
__device__ __forceinline__ double ys_pair_factor(double d2, double c, double S, int si,
                                                 const double* __restrict__ T0) {
  const double y = rsqrt_fast(d2);
  const double r = __dmul_rn(d2, y);
  const double z = fma(r, -c, S);
  const int k = __double2loint(z);
  const double f = fma(r, -c, (double)(si - k));
  constexpr double a1 = 0x1.62e42fefa39efp-12;   // ln2 / 2048
  constexpr double a2 = a1 * a1 / 2.0;
  constexpr double a3 = a1 * a1 * a1 / 6.0;
  double p = fma(a3, f, a2);
  p = fma(p, f, a1);
  p = fma(p, f, 1.0);
  return __dmul_rn(__dmul_rn(T0[k], p), y);
}

// The near field's YS factor with s = 0: k = rint(-c r) <= 0; the index is
// clamped into [-2048, 0] for the zero-charge padding records far away
// (their factor is then finite garbage times q = 0).
__device__ __forceinline__ double ys_pair_factor_near(double d2, double c,
                                                      const double* __restrict__ T0) {
  const double kMagic = 6755399441055744.0;   // 1.5 * 2^52
  const double y = rsqrt_fast(d2);
  const double r = __dmul_rn(d2, y);
  const double z = fma(r, -c, kMagic);
  const int kr = __double2loint(z);
  const int k = -(int)umin((unsigned)(-kr), (unsigned)kExp2WK);   // [-2048, 0]
  const double f = fma(r, -c, (double)(-kr));   // magic - z = -k, via I2F (see ys_pair_factor)
  constexpr double a1 = 0x1.62e42fefa39efp-12;   // ln2 / 2048
  constexpr double a2 = a1 * a1 / 2.0;
  constexpr double a3 = a1 * a1 * a1 / 6.0;
  double p = fma(a3, f, a2);
  p = fma(p, f, a1);
  p = fma(p, f, 1.0);
  return __dmul_rn(__dmul_rn(T0[k], p), y);
}

__device__ __forceinline__ YsState ys_state(double tx, double ty, double tz, double cx, double cy,
                                            double cz, double c, const double* __restrict__ T0,
                                            bool& ok) {
  const double kMagic = 6755399441055744.0;   // 1.5 * 2^52
  const double dx = tx - cx, dy = ty - cy, dz = tz - cz;
  const double u = c * sqrt(fma(dx, dx, fma(dy, dy, dz * dz)));
  ok = u < 0x1p30;
  const double sd = ok ? rint(u) : 0.0;
  YsState st;
  st.S = kMagic + sd;
  st.si = (int)sd;
  // 2^(-s/2048) = 2^(-m) T[-j], s = 2048 m + j, 0 <= j < 2048
  const long long si = (long long)sd;
  const int j = (int)(si & 2047);
  const long long m = si >> 11;
  st.E = m > 1100 ? 0.0 : ldexp(T0[-j], -(int)m);
  return st;
}

// One cluster's FAST Yukawa far-field sum for one target, generic exponential,
// moments from global memory: the YS kernel's rare fallback, kept out of line
// so the hot loop stays small.
template <int M>
__device__ __noinline__ double far_cluster_generic(const double* __restrict__ row,
                                                   const double* __restrict__ pts, double tx,
                                                   double ty, double tz, YukawaK yk) {
  double part = 0.0;
  for (int k1 = 0; k1 < M; ++k1) {
    const double dx = tx - pts[k1];
    for (int k2 = 0; k2 < M; ++k2) {
      const double dy = ty - pts[M + k2];
      const double dxy = fma(dy, dy, dx * dx);
      for (int k3 = 0; k3 < M; ++k3) {
        const double dz = tz - pts[2 * M + k3];
        part = pair_acc<1, 2>(part, row[(k1 * M + k2) * M + k3], fma(dz, dz, dxy), yk);
      }
    }
  }
  return part;
}

template <int KIND, int M, int KU, int FORM, bool PAR = false, bool DY = false, bool YS = false>
__device__ __forceinline__ void far_packed_item(const EvalArgs& a, const int4 it,
                                                const int32_t* poff, double* wsm, int lane,
                                                const double* __restrict__ T0 = nullptr) {
  using SM = FarSmem<M>;
  double* dys = wsm + SM::kWarp + lane;   // DY slots: dys[(k2 * 2 + t) * 32]
  FarHdr* H = reinterpret_cast<FarHdr*>(wsm);
  const LaneTargets L = lane_targets(it, a, poff, lane);
  const double tx[2] = {a.tx[L.i0], a.tx[L.i1]};
  const double ty[2] = {a.ty[L.i0], a.ty[L.i1]};
  const double tz[2] = {a.tz[L.i0], a.tz[L.i1]};
  double acc[2] = {0.0, 0.0};
  if (PAR && !a.par_first) {   // later source group: continue the running out
    acc[0] = a.far_out[L.i0];
    acc[1] = a.far_out[L.i1];
  }

  // segment list ranges (warp-uniform) into the header
  int maxlen = 0, mylen = 0;
  __syncwarp();
  if (lane < kGMax) {
    int e0 = 0, len = 0;
    if (lane < it.w) {
      const int64_t b = it.z + lane;
      e0 = a.a_ptr[b * a.G + a.g_lo];
      len = a.a_ptr[b * a.G + a.g_hi] - e0;
    }
    H->e0[lane] = e0;
    H->len[lane] = len;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kGMax; ++k) maxlen = max(maxlen, H->len[k]);
  mylen = H->len[L.g];
  const double* mpts = wsm + SM::kHdr + L.g * SM::kSeg;   // this lane's segment region
  const double* mslab = mpts + SM::kPts;

  for (int e = 0; e < maxlen; ++e) {
    __syncwarp();
    // this step's cluster of every segment: header row pointers, proxy points
    if (lane < kGMax) {
      const double* row = nullptr;
      if (e < H->len[lane]) {
        const EvalCluster* c = a.clusters + a.a_idx[H->e0[lane] + e];
        row = a.moments + (size_t)c->mrow * a.mstride;
      }
      H->row[lane] = row;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kGMax; ++k) {
      if (H->row[k] != nullptr) {
        const EvalCluster* c = a.clusters + a.a_idx[H->e0[k] + e];
        double* seg = wsm + SM::kHdr + k * SM::kSeg;
        for (int i = lane; i < SM::kPts; i += 32) {
          const int d = i / M, kk = i - d * M;
          seg[i] = cheb_point_dev(a.degree, kk, c->lo[d], c->hi[d], a.s_nodes);
        }
      }
    }
    far_stage_slab<M>(wsm, H, 0, lane);
    const bool act = e < mylen;
    double part[2] = {0.0, 0.0};
    bool slow[2] = {false, false};   // PAR, Coulomb: an operand left the fast path
    __syncwarp();   // proxy points (plain stores) visible to the warp
    YsState ys[2];
    bool use_ys = false;
    if constexpr (YS) {
      // bounds from the lane's OWN segment's staged proxy points (current, or
      // stale for an idle segment -- its results are discarded, but its table
      // index must stay in range too): box [p[M-1], p[0]] per axis
      const double ex = mpts[0] - mpts[M - 1], ey = mpts[M] - mpts[2 * M - 1],
                   ez = mpts[2 * M] - mpts[3 * M - 1];
      const double hd = 0.5 * sqrt(fma(ex, ex, fma(ey, ey, ez * ez)));
      const double cx = 0.5 * (mpts[0] + mpts[M - 1]);
      const double cy = 0.5 * (mpts[M] + mpts[2 * M - 1]);
      const double cz = 0.5 * (mpts[2 * M] + mpts[3 * M - 1]);
      bool ok0, ok1;
      ys[0] = ys_state(tx[0], ty[0], tz[0], cx, cy, cz, a.yk.c2, T0, ok0);
      ys[1] = ys_state(tx[1], ty[1], tz[1], cx, cy, cz, a.yk.c2, T0, ok1);
      use_ys = __all_sync(0xffffffffu, ok0 && ok1 && a.yk.c2 * hd + 2.0 <= (double)kExp2WK);
      if (!use_ys) {
        // rare: a cluster too large for the table at this kappa -- the
        // generic exponential, straight from the moment row in global memory
        cp_async_wait<0>();
        __syncwarp();
        const double* row = H->row[L.g];
#pragma unroll 1
        for (int t = 0; t < 2; ++t)
          part[t] = act ? far_cluster_generic<M>(row, mpts, tx[t], ty[t], tz[t], a.yk) : 0.0;
#pragma unroll
        for (int t = 0; t < 2; ++t) acc[t] = act ? __dadd_rn(acc[t], part[t]) : acc[t];
        continue;
      }
    }
    double dz2[2][M];
#pragma unroll
    for (int k3 = 0; k3 < M; ++k3) {
      const double p3 = mpts[2 * M + k3];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double dz = __dsub_rn(tz[t], p3);
        dz2[t][k3] = __dmul_rn(dz, dz);
      }
    }
    if constexpr (DY) {
      for (int k2 = 0; k2 < M; ++k2) {
        const double p2 = mpts[M + k2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const double dy = __dsub_rn(ty[t], p2);
          dys[(k2 * 2 + t) * 32] = __dmul_rn(dy, dy);
        }
      }
    }
    for (int k1 = 0; k1 < M; ++k1) {
      if (k1 + 1 < M) {
        far_stage_slab<M>(wsm, H, k1 + 1, lane);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const double p1 = mpts[k1];
      double dx2[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double dx = __dsub_rn(tx[t], p1);
        dx2[t] = __dmul_rn(dx, dx);
      }
      const double* qr = mslab + (k1 & 1) * SM::kSlab;
#pragma unroll KU
      for (int k2 = 0; k2 < M; ++k2, qr += M) {
        const double p2 = mpts[M + k2];
        double dxy2[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if constexpr (DY) {
            dxy2[t] = __dadd_rn(dx2[t], dys[(k2 * 2 + t) * 32]);
          } else {
            const double dy = __dsub_rn(ty[t], p2);
            dxy2[t] = PAR ? __dadd_rn(dx2[t], __dmul_rn(dy, dy)) : fma(dy, dy, dx2[t]);
          }
        }
#pragma unroll
        for (int k3 = 0; k3 < M; ++k3) {
          const double qv = qr[k3];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const double d2 = __dadd_rn(dxy2[t], dz2[t][k3]);
            if (PAR && KIND == 0) {
              bool ok;
              part[t] = __dadd_rn(part[t], coulomb_parity_fp(qv, d2, ok));
              slow[t] |= !ok;
            } else if (PAR) {
              part[t] = __dadd_rn(part[t], parity_term<KIND>(qv, d2, a.kappa));
            } else if (YS) {
              part[t] = fma(qv, ys_pair_factor(d2, a.yk.c2, ys[t].S, ys[t].si, T0), part[t]);
            } else {
              part[t] = pair_acc<KIND, FORM>(part[t], qv, d2, a.yk);
            }
          }
        }
      }
      __syncwarp();
    }
    if (PAR && KIND == 0 && __any_sync(0xffffffffu, slow[0] || slow[1])) {
      // rare: redo this cluster's sum with the intrinsics (moments from the
      // row in global memory -- the staged slabs are gone)
      const double* row = H->row[L.g];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (!(slow[t] && act)) continue;
        double p = 0.0;
        int qi = 0;
        for (int k1 = 0; k1 < M; ++k1) {
          const double dx = __dsub_rn(tx[t], mpts[k1]);
          for (int k2 = 0; k2 < M; ++k2) {
            const double dy = __dsub_rn(ty[t], mpts[M + k2]);
            const double dxy = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            for (int k3 = 0; k3 < M; ++k3) {
              const double dz = __dsub_rn(tz[t], mpts[2 * M + k3]);
              const double d2 = __dadd_rn(dxy, __dmul_rn(dz, dz));
              p = __dadd_rn(p, parity_term<KIND>(row[qi++], d2, a.kappa));
            }
          }
        }
        part[t] = p;
      }
    }
    if (YS) {
#pragma unroll
      for (int t = 0; t < 2; ++t) part[t] = __dmul_rn(part[t], ys[t].E);
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) acc[t] = act ? __dadd_rn(acc[t], part[t]) : acc[t];
  }
  if (L.v0) a.far_out[L.i0] = acc[0];
  if (L.v1) a.far_out[L.i1] = acc[1];
}

template <int KIND, int M, int MINB, int KU, int FORM, bool PAR = false, bool DY = false,
          bool YS = false>
__global__ void __launch_bounds__(kWarps * 32, MINB)
k_far_packed(EvalArgs a, const int4* __restrict__ items, int n_items, const int32_t* poff,
             int* counter) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kPerWarp = FarSmem<M>::kWarp + (DY ? FarSmem<M>::kDy : 0);
  double* wsm = smem + warp * kPerWarp;
  const double* T0 = nullptr;
  if constexpr (YS) {   // the shifted-exp table behind the warps' regions
    double* tab = smem + kWarps * kPerWarp;
    for (int i = threadIdx.x; i < 2 * kExp2WK + 1; i += blockDim.x) tab[i] = kExp2W[i];
    // proxy points of never-used segments: a point box (bounded table index)
    for (int i = threadIdx.x; i < kWarps * kPerWarp; i += blockDim.x) smem[i] = 0.0;
    __syncthreads();
    T0 = tab + kExp2WK;
  }
  for (int item = next_item(counter); item < n_items; item = next_item(counter))
    far_packed_item<KIND, M, KU, FORM, PAR, DY, YS>(a, items[item], poff, wsm, lane, T0);
}

// ---------------------------------------------------------------------------
// Near field.
template <int CH>
struct NearSmem {
  // [segment][buffer][CH] packed sources; +1 record between segments
  static constexpr int kSeg = 2 * CH + 1;
  static constexpr int kWarp = kGMax * kSeg;
};

#ifndef BLTC_NEAR_UNROLL
#define BLTC_NEAR_UNROLL 4
#endif
constexpr int kNearUnroll = BLTC_NEAR_UNROLL;   // pragma arguments are not macro-expanded
#ifndef BLTC_FOLD_CHUNKS
#define BLTC_FOLD_CHUNKS 4
#endif
// FAST near field: chunk partials are Neumaier-folded into (acc, comp) every
// kFoldChunks chunks of 32 sources (C4 near 206.0 ms folding every chunk,
// 204.3 every 2, 203.4 every 4, 202.7 every 8)
constexpr int kFoldChunks = BLTC_FOLD_CHUNKS;
// A non-negative double (2^-126 <= x < 2^128) as a float from its high
// word alone, truncated to 20 mantissa bits (so <= x, within 2^-20):
// integer-pipe work (LEA), no FP64 instruction.  CLAMP: smaller x clamp up
// to 2^-126 (an over-estimate).
template <bool CLAMP>
__device__ __forceinline__ float hi_float(double x) {
  int h = __double2hiint(x);
  if (CLAMP) h = max(h, 0x38100000);
  return __int_as_float((h - 0x38000000) << 3);
}

// STRICT's near-field mass sum_j |q_j| f_j (f = the kernel factor) per
// target, variants (BLTC_ABS, measured in DESIGN.md 5.1):
//   1: FP64, one more DFMA per pair (|q| f)
//   2: FP32 on the integer / FP32 pipes: |q| from its high word (clamped),
//      f from the rsqrt seed's high word (2^-20), one FFMA per pair
//   3: FP32 sum of f from the seed's high word (one LEA + FADD per pair),
//      times max |q| at the end
// 2 and 3 need f in the float range: coordinates below 2^50 (guarded,
// strict.cu) and zero-charge padding records at 2^60.
template <int KIND, int CH, bool MASKED, int FORM, int ABS = 0, bool YS = false>
__device__ __forceinline__ void near_chunk(double (&part)[2], double (&apart)[2],
                                           float (&fpart)[2], const double4* src,
                                           const double (&tx)[2], const double (&ty)[2],
                                           const double (&tz)[2], const YukawaK& yk,
                                           const double* __restrict__ T0 = nullptr) {
  const long long tb = __double_as_longlong(kSingularSq);   // d2 >= 0: bit order = value order
#pragma unroll kNearUnroll
  for (int j = 0; j < CH; ++j) {
    const double4 s = src[j];
    const float qa = ABS == 2 ? hi_float<true>(fabs(s.w)) : 0.0f;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double dx = __dsub_rn(tx[t], s.x);
      const double dy = __dsub_rn(ty[t], s.y);
      const double dz = __dsub_rn(tz[t], s.z);
      double d2, q;
      bool ok = true;
      if (MASKED) {
        // d2 + 1e-300: exactly d2 for every non-singular pair, never 0, so
        // only the charge needs the select (excluded pairs add 0 * finite)
        d2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, 1e-300)));
        ok = __double_as_longlong(d2) >= tb;
        q = ok ? s.w : 0.0;
      } else {
        d2 = fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx)));
        q = s.w;
      }
      if (YS) {   // Yukawa, shifted-exp table with s = 0 (the batch's flag holds)
        const double f = ys_pair_factor_near(d2, yk.c2, T0);
        part[t] = fma(q, f, part[t]);
        if (ABS == 1) apart[t] = fma(fabs(q), f, apart[t]);
      } else if (ABS == 1) {
        const double f = pair_factor<KIND>(d2, yk);
        part[t] = fma(q, f, part[t]);
        apart[t] = fma(fabs(q), f, apart[t]);
      } else if (ABS >= 2) {
        double y0;   // the rsqrt seed (2^-20): its high word is the mass estimate
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d2));
        // Yukawa: exp(-kappa r) / r <= 1 / r, the Coulomb mass bounds it
        const float fa = hi_float<false>(y0);
        if (ABS == 2) fpart[t] = fmaf(ok ? qa : 0.0f, fa, fpart[t]);
        else fpart[t] += ok ? fa : 0.0f;
        part[t] = pair_acc<KIND, 2>(part[t], q, d2, yk);
      } else {
        part[t] = pair_acc<KIND, FORM>(part[t], q, d2, yk);
      }
    }
  }
}

// PARITY: the reference's _direct_tile pair by pair -- d2 unfused, pairs with
// d2 < 1e-28 skipped, Neumaier into (acc, comp) (engine.py:166-213).  The
// zero-charge padding records add +0 exactly (acc and comp are never -0).
// FP: Coulomb terms on the intrinsics' fast paths; the caller replays the
// chunk with FP = false for the (rare) lanes that report `slow`.
template <int KIND, int CH, bool MASKED, bool FP = false>
__device__ __forceinline__ void near_chunk_parity(double (&acc)[2], double (&comp)[2],
                                                  const double4* src, const double (&tx)[2],
                                                  const double (&ty)[2],
                                                  const double (&tz)[2], double kappa,
                                                  bool (&slow)[2]) {
  const long long tb = __double_as_longlong(kSingularSq);
#pragma unroll 2
  for (int j = 0; j < CH; ++j) {
    const double4 s = src[j];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double dx = __dsub_rn(tx[t], s.x);
      const double dy = __dsub_rn(ty[t], s.y);
      const double dz = __dsub_rn(tz[t], s.z);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      const bool ok = !MASKED || __double_as_longlong(d2) >= tb;
      double term;
      if (FP && KIND == 0) {
        bool fast;
        term = coulomb_parity_fp(s.w, ok ? d2 : 1.0, fast);
        slow[t] |= ok && !fast;
      } else {
        term = parity_term<KIND>(s.w, ok ? d2 : 1.0, kappa);
      }
      const double sum = __dadd_rn(acc[t], term);
      const bool big = fabs(acc[t]) >= fabs(term);
      const double hi = big ? acc[t] : term, lo = big ? term : acc[t];
      const double c2 = __dadd_rn(comp[t], __dadd_rn(__dsub_rn(hi, sum), lo));
      acc[t] = ok ? sum : acc[t];
      comp[t] = ok ? c2 : comp[t];
    }
  }
}

// One segment's source stream: the sources of its direct list, cluster
// after cluster in list order.  Warp-uniform state: list entry e, offset o
// within that cluster, the cluster's (start, count, mask flag) and the next
// entry's, loaded one advance ahead so that staging a chunk needs no
// dependent loads in the common case.
struct Stream {
  int e0, len;        // list segment [e0, e0 + len)
  int e, o;           // position
  int cs, cn, ns, nn; // current / next cluster: first source, count
  bool cm, nm;        // current / next: singular pairs possible
};

__device__ __forceinline__ void stream_entry(const EvalArgs& a, const uint8_t* dmask, int ent,
                                             int* start, int* count, bool* m) {
  const EvalCluster& c = a.clusters[a.d_idx[ent]];
  *start = c.start;
  *count = c.stop - c.start;
  *m = dmask[ent] != 0;
}

__device__ __forceinline__ void stream_init(const EvalArgs& a, const uint8_t* dmask, Stream& S,
                                            int e0, int len) {
  S.e0 = e0;
  S.len = len;
  S.e = 0;
  S.o = 0;
  S.cs = S.cn = S.ns = S.nn = 0;
  S.cm = S.nm = false;
  if (len > 0) stream_entry(a, dmask, e0, &S.cs, &S.cn, &S.cm);
  if (len > 1) stream_entry(a, dmask, e0 + 1, &S.ns, &S.nn, &S.nm);
}

// Source index of record o + r0 of the stream (-1: past its end); need_mask:
// the record may form singular pairs.
__device__ __forceinline__ int stream_src(const EvalArgs& a, const uint8_t* dmask,
                                          const Stream& S, int r0, bool& need_mask) {
  need_mask = false;
  int src = -1;
  if (S.e < S.len) {
    const int r = S.o + r0;
    if (r < S.cn) {
      src = S.cs + r;
      need_mask = S.cm;
    } else if (r - S.cn < S.nn) {
      src = S.ns + (r - S.cn);
      need_mask = S.nm;
    } else {
      // the chunk spans more than two clusters (small clusters): walk
      int rr = r - S.cn - S.nn;
      for (int e = S.e + 2; e < S.len; ++e) {
        int st, n;
        bool m;
        stream_entry(a, dmask, S.e0 + e, &st, &n, &m);
        if (rr < n) {
          src = st + rr;
          need_mask = m;
          break;
        }
        rr -= n;
      }
    }
  }
  return src;
}

// Stage record o + r of the stream into dst[r]; returns whether it may form
// singular pairs.
__device__ __forceinline__ bool stream_stage(const EvalArgs& a, const uint8_t* dmask,
                                             const Stream& S, double4* dst, int r0) {
  bool need_mask;
  const int src = stream_src(a, dmask, S, r0, need_mask);
  if (src >= 0) {
    const double4* sp = a.src4 + src;
    cp_async16(dst + r0, sp);
    cp_async16(reinterpret_cast<char*>(dst + r0) + 16, reinterpret_cast<const char*>(sp) + 16);
  } else {
    dst[r0] = make_double4(0x1p60, 0x1p60, 0x1p60, 0.0);   // contributes exactly 0
  }
  return need_mask;
}

template <int CH>
__device__ __forceinline__ void stream_advance(const EvalArgs& a, const uint8_t* dmask,
                                               Stream& S) {
  S.o += CH;
  while (S.e < S.len && S.o >= S.cn) {
    S.o -= S.cn;
    ++S.e;
    S.cs = S.ns;
    S.cn = S.nn;
    S.cm = S.nm;
    S.nn = 0;
    if (S.e + 1 < S.len) stream_entry(a, dmask, S.e0 + S.e + 1, &S.ns, &S.nn, &S.nm);
  }
}

// Stage the next chunk of every live segment into buffer `buf`.
template <int CH>
__device__ __forceinline__ bool near_stage(const EvalArgs& a, const uint8_t* dmask,
                                           Stream (&S)[kGMax], double4* wsm, int buf,
                                           int lane) {
  bool need_mask = false;
#pragma unroll
  for (int k = 0; k < kGMax; ++k) {
    double4* dst = wsm + k * NearSmem<CH>::kSeg + buf * CH;
#pragma unroll
    for (int r = 0; r < CH; r += 32) need_mask |= stream_stage(a, dmask, S[k], dst, r + lane);
    stream_advance<CH>(a, dmask, S[k]);
  }
  cp_async_commit();
  return __any_sync(0xffffffffu, need_mask);
}

// BULK: the same chunk staged by the TMA engine.  Each segment's 32 records
// are runs of consecutive sources (a cluster's tail, the next cluster's
// head, ...): the first lane of each run issues one cp.async.bulk of the
// whole run; lane 0 first arms the buffer's mbarrier with the chunk's byte
// count; past-the-end records are written as zero-charge padding.
template <int CH>
__device__ __forceinline__ bool near_stage_bulk(const EvalArgs& a, const uint8_t* dmask,
                                                Stream (&S)[kGMax], double4* wsm, int buf,
                                                int lane, uint64_t* bar) {
  static_assert(CH == 32, "bulk staging: one record per lane");
  bool need_mask = false;
  int src[kGMax];
  unsigned total = 0;
#pragma unroll
  for (int k = 0; k < kGMax; ++k) {
    bool m;
    src[k] = stream_src(a, dmask, S[k], lane, m);
    need_mask |= m;
    total += 32u * __popc(__ballot_sync(0xffffffffu, src[k] >= 0));
    stream_advance<CH>(a, dmask, S[k]);
  }
  if (lane == 0) mbar_arrive_expect_tx(bar, total * 1u);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < kGMax; ++k) {
    double4* dst = wsm + k * NearSmem<CH>::kSeg + buf * CH;
    const int prev = __shfl_up_sync(0xffffffffu, src[k], 1);
    const bool valid = src[k] >= 0;
    const bool lead = valid && (lane == 0 || prev != src[k] - 1);
    const unsigned ends = __ballot_sync(0xffffffffu, lead || !valid);
    if (lead) {
      const unsigned later = lane == 31 ? 0u : ends >> (lane + 1);
      const int len = later ? __ffs(later) : 32 - lane;
      bulk_g2s(dst + lane, a.src4 + src[k], 32u * len, bar);
    } else if (!valid) {
      dst[lane] = make_double4(0x1p60, 0x1p60, 0x1p60, 0.0);   // contributes exactly 0
    }
  }
  return __any_sync(0xffffffffu, need_mask);
}

// PAR: the direct sums continue the far-field value of each target with
// per-pair Neumaier compensation, out = acc + carry at the end (engine.py:
// 302-312, 335); over several source groups one pass per group, (acc, carry)
// handed from pass to pass (decomp.py:437-454).
template <int KIND, int CH, int FORM, bool PAR = false, bool BULK = false, int ABS = 0,
          bool YS = false>
__device__ __forceinline__ void near_packed_item(const EvalArgs& a, const int4 it,
                                                 const int32_t* poff, const uint8_t* dmask,
                                                 double4* wsm, int lane, uint64_t* bar,
                                                 unsigned& phase,
                                                 const double* __restrict__ T0 = nullptr) {
  const LaneTargets L = lane_targets(it, a, poff, lane);
  const double tx[2] = {a.tx[L.i0], a.tx[L.i1]};
  const double ty[2] = {a.ty[L.i0], a.ty[L.i1]};
  const double tz[2] = {a.tz[L.i0], a.tz[L.i1]};
  double acc[2] = {0.0, 0.0}, comp[2] = {0.0, 0.0};
  if (PAR) {
    acc[0] = a.far_out[L.i0];
    acc[1] = a.far_out[L.i1];
    if (!a.par_first) {
      comp[0] = a.carry[L.i0];
      comp[1] = a.carry[L.i1];
    }
  }

  Stream S[kGMax];
#pragma unroll
  for (int k = 0; k < kGMax; ++k) {
    int e0 = 0, len = 0;
    if (k < it.w) {
      const int64_t b = it.z + k;
      e0 = a.d_ptr[b * a.G + a.g_lo];
      len = a.d_ptr[b * a.G + a.g_hi] - e0;
    }
    stream_init(a, dmask, S[k], e0, len);
  }
  const double4* mine = wsm + L.g * NearSmem<CH>::kSeg;
  double npart[2] = {0.0, 0.0};   // FAST: partial sum over the last chunks
  double apart[2] = {0.0, 0.0};   // ABS 1 (STRICT): sum of |q f| (FP64)
  float fpart[2] = {0.0f, 0.0f};  // ABS 2 / 3: the last chunks' mass in FP32
  double aacc[2] = {0.0, 0.0};    // ABS 2 / 3: the folded FP32 partials
  int nchunk = 0;
  bool live = false;
#pragma unroll
  for (int k = 0; k < kGMax; ++k) live |= S[k].e < S[k].len;
  if (live) {
    __syncwarp();
    bool masked = BULK ? near_stage_bulk<CH>(a, dmask, S, wsm, 0, lane, bar)
                       : near_stage<CH>(a, dmask, S, wsm, 0, lane);
    for (int buf = 0;; buf ^= 1) {
      bool more = false;
#pragma unroll
      for (int k = 0; k < kGMax; ++k) more |= S[k].e < S[k].len;
      bool masked_next = false;
      if constexpr (BULK) {
        if (more) masked_next = near_stage_bulk<CH>(a, dmask, S, wsm, buf ^ 1, lane, bar + (buf ^ 1));
        mbar_wait(bar + buf, (phase >> buf) & 1u);
        phase ^= 1u << buf;
      } else if (more) {
        masked_next = near_stage<CH>(a, dmask, S, wsm, buf ^ 1, lane);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      if constexpr (PAR) {
        const double acc0[2] = {acc[0], acc[1]}, comp0[2] = {comp[0], comp[1]};
        bool slow[2] = {false, false};
        if (masked)
          near_chunk_parity<KIND, CH, true, KIND == 0>(acc, comp, mine + buf * CH, tx, ty, tz,
                                                       a.kappa, slow);
        else
          near_chunk_parity<KIND, CH, false, KIND == 0>(acc, comp, mine + buf * CH, tx, ty, tz,
                                                        a.kappa, slow);
        if (KIND == 0 && __any_sync(0xffffffffu, slow[0] || slow[1])) {
          // rare: replay the chunk with the intrinsics from its starting state
          double acc1[2] = {acc0[0], acc0[1]}, comp1[2] = {comp0[0], comp0[1]};
          bool unused[2] = {false, false};
          if (masked)
            near_chunk_parity<KIND, CH, true>(acc1, comp1, mine + buf * CH, tx, ty, tz,
                                              a.kappa, unused);
          else
            near_chunk_parity<KIND, CH, false>(acc1, comp1, mine + buf * CH, tx, ty, tz,
                                               a.kappa, unused);
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (slow[t]) {
              acc[t] = acc1[t];
              comp[t] = comp1[t];
            }
        }
      } else {
        if (masked)
          near_chunk<KIND, CH, true, FORM, ABS, YS>(npart, apart, fpart, mine + buf * CH, tx,
                                                    ty, tz, a.yk, T0);
        else
          near_chunk<KIND, CH, false, FORM, ABS, YS>(npart, apart, fpart, mine + buf * CH, tx,
                                                     ty, tz, a.yk, T0);
        if ((++nchunk & (kFoldChunks - 1)) == 0 || !more) {   // fold every kFoldChunks chunks
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            neumaier(acc[t], comp[t], npart[t]);
            npart[t] = 0.0;
            if (ABS >= 2) {
              aacc[t] += (double)fpart[t];
              fpart[t] = 0.0f;
            }
          }
        }
      }
      __syncwarp();
      if (!more) break;
      masked = masked_next;
    }
  }
  // approximations first, then the compensated direct sums on top
  // (engine.py:302-312, 335)
  if (PAR) {
    if (!a.par_last) {   // more source groups follow: keep (out, carry) apart
      if (L.v0) {
        a.far_out[L.i0] = acc[0];
        a.carry[L.i0] = comp[0];
      }
      if (L.v1) {
        a.far_out[L.i1] = acc[1];
        a.carry[L.i1] = comp[1];
      }
      return;
    }
    if (L.v0) a.out[L.i0] = __dadd_rn(acc[0], comp[0]);
    if (L.v1) a.out[L.i1] = __dadd_rn(acc[1], comp[1]);
    return;
  }
  if (ABS) {
    // ABS 2 / 3: truncated high words (2^-19 per term) and FP32 partials of
    // <= 4 x 32 positive terms (< 2^-16 relative): covered by 2^-12
    // (ABS 3: strict.cu multiplies by max |q|)
    const double sc = ABS == 1 ? 1.0 : 1.0 + 0x1p-12;
    if (L.v0) a.absum[L.i0] = (ABS == 1 ? apart[0] : aacc[0]) * sc;
    if (L.v1) a.absum[L.i1] = (ABS == 1 ? apart[1] : aacc[1]) * sc;
  }
  if (L.v0) {
    double total = acc[0], cmp = comp[0];
    neumaier(total, cmp, a.far_out[L.i0]);
    a.out[L.i0] = __dadd_rn(total, cmp);
  }
  if (L.v1) {
    double total = acc[1], cmp = comp[1];
    neumaier(total, cmp, a.far_out[L.i1]);
    a.out[L.i1] = __dadd_rn(total, cmp);
  }
}

template <int KIND, int CH, int MINB, int FORM, bool PAR = false, bool BULK = false,
          int ABS = 0, bool YS = false>
__global__ void __launch_bounds__(kWarps * 32, MINB)
k_near_packed(EvalArgs a, const int4* __restrict__ items, int n_items, const int32_t* poff,
              const uint8_t* dmask, const uint8_t* bys, int* counter) {
  extern __shared__ double4 nsmem[];
  __shared__ uint64_t nbar[kWarps][2];   // BULK: one mbarrier per staging buffer
  double4* smem = nsmem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double4* wsm = smem + warp * NearSmem<CH>::kWarp;
  if (BULK && lane == 0) {
    mbar_init(&nbar[warp][0], 1);
    mbar_init(&nbar[warp][1], 1);
  }
  const double* T0 = nullptr;
  if constexpr (YS) {   // the shifted-exp table behind the warps' staging buffers
    double* tab = reinterpret_cast<double*>(smem + kWarps * NearSmem<CH>::kWarp);
    for (int i = threadIdx.x; i < 2 * kExp2WK + 1; i += blockDim.x) tab[i] = kExp2W[i];
    __syncthreads();
    T0 = tab + kExp2WK;
  }
  __syncwarp();
  unsigned phase = 0;
  for (int item = next_item(counter); item < n_items; item = next_item(counter)) {
    const int4 it = items[item];
    if constexpr (YS) {
      // the item's batches all within the table's reach: the YS pair loop
      bool ok = true;
#pragma unroll
      for (int k = 0; k < kGMax; ++k) ok &= k >= it.w || bys[it.z + k] != 0;
      if (ok) {
        near_packed_item<KIND, CH, FORM, PAR, BULK, ABS, true>(a, it, poff, dmask, wsm, lane,
                                                             nbar[warp], phase, T0);
        continue;
      }
    }
    near_packed_item<KIND, CH, FORM, PAR, BULK, ABS>(a, it, poff, dmask, wsm, lane, nbar[warp],
                                                     phase);
  }
}

// ---------------------------------------------------------------------------
// Tuning switches for measurements (BLTC_FAR_UNROLL=1|3, BLTC_PFORM=0|2).
int tune_far_unroll(int kind) {
  const char* e = std::getenv("BLTC_FAR_UNROLL");
  // Coulomb: 3 rows per step, -2% far time at C4 (measured)
  return e ? std::atoi(e) : (kind == 0 ? 3 : 1);
}
int tune_near_bulk() {
  const char* e = std::getenv("BLTC_NEAR_BULK");
  return e ? std::atoi(e) : 0;
}
int tune_far_dy() {
  const char* e = std::getenv("BLTC_FAR_DY");
  return e ? std::atoi(e) : 1;   // dy^2 per (target, k2) in shared memory: -0.7% far (measured)
}
int tune_yshift() {
  const char* e = std::getenv("BLTC_YSHIFT");
  return e ? std::atoi(e) : 1;
}
int tune_form() {
  const char* e = std::getenv("BLTC_PFORM");
  return e ? std::atoi(e) : 2;   // FORM 2: -0.9% far, -1.5% near at C4 (measured)
}


template <typename K>
int persistent_grid(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  BLTC_CUDA(cudaGetDevice(&dev));
  BLTC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  BLTC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  return sms * (per_sm > 0 ? per_sm : 1);
}

template <int KIND, int M, int KU = 1, int FORM = 0, int MINB = 2, bool PAR = false,
          bool DY = false, bool YS = false>
void far_packed_launch(const EvalArgs& a, const PackedItems& it, int* counter, cudaStream_t st) {
  const size_t smem =
      sizeof(double) * (kWarps * (FarSmem<M>::kWarp + (DY ? FarSmem<M>::kDy : 0)) +
                        (YS ? 2 * kExp2WK + 1 : 0));
  auto kern = k_far_packed<KIND, M, MINB, KU, FORM, PAR, DY, YS>;
  BLTC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = persistent_grid(kern, kWarps * 32, smem);
  kern<<<grid, kWarps * 32, smem, st>>>(a, it.items_far, it.n_items, it.poff, counter);
  BLTC_LAUNCH_CHECK();
}

template <int KIND>
bool far_packed_dispatch_parity(const EvalArgs& a, const PackedItems& it, int* counter,
                                cudaStream_t st) {
  switch (a.degree + 1) {
#define BLTC_PAR_CASE(MM) \
    case MM: far_packed_launch<KIND, MM, 1, 0, 2, true>(a, it, counter, st); return true;
    case 9:
      // the benchmark degree: one CTA per SM with the full register file and
      // k2 unrolled by 3 -- the IEEE sqrt / division chains want ILP more
      // than warps (C4 far 2151 -> 2054 ms; 2 CTAs per SM spill at 128 regs)
      // dy^2 per (target, k2) in shared memory (the same rounded products):
      // 2053 -> 2034 ms; k2 x9: 2482 ms
      far_packed_launch<KIND, 9, 3, 0, 1, true, true>(a, it, counter, st);
      return true;
    BLTC_PAR_CASE(2) BLTC_PAR_CASE(3) BLTC_PAR_CASE(4) BLTC_PAR_CASE(5) BLTC_PAR_CASE(6)
    BLTC_PAR_CASE(7) BLTC_PAR_CASE(8) BLTC_PAR_CASE(10) BLTC_PAR_CASE(11)
    BLTC_PAR_CASE(12) BLTC_PAR_CASE(13)
#undef BLTC_PAR_CASE
    default: return false;
  }
}

template <int KIND>
bool far_packed_dispatch(const EvalArgs& a, const PackedItems& it, int* counter,
                         cudaStream_t st) {
  switch (a.degree + 1) {
#define BLTC_FAST_CASE(MM) \
    case MM: far_packed_launch<KIND, MM>(a, it, counter, st); return true;
    BLTC_FAST_CASE(2) BLTC_FAST_CASE(3) BLTC_FAST_CASE(4) BLTC_FAST_CASE(5) BLTC_FAST_CASE(6)
    BLTC_FAST_CASE(7) BLTC_FAST_CASE(8) BLTC_FAST_CASE(10)
    BLTC_FAST_CASE(12) BLTC_FAST_CASE(13)
    case 11:
      // C5's degree: FORM 2 (C5 far 8382 -> 8282 ms; k2 x3 with one CTA per
      // SM 8292, one CTA per SM alone 8700)
      if (tune_form() == 2) far_packed_launch<KIND, 11, 1, 2>(a, it, counter, st);
      else far_packed_launch<KIND, 11>(a, it, counter, st);
      return true;
#undef BLTC_FAST_CASE
    case 9:
      // tuned for the benchmark degree: k2 unrolled by 3, FORM 2 (measured)
      if (tune_form() != 2) far_packed_launch<KIND, 9, 1, 0>(a, it, counter, st);
      else if (KIND == 1 && tune_yshift())   // Yukawa, shifted exponential (YS)
        far_packed_launch<KIND, 9, 3, 2, 1, false, false, true>(a, it, counter, st);
      else if (KIND == 1)   // Yukawa: one CTA per SM, full register file (C3 far -4%; x9 +10%)
        far_packed_launch<KIND, 9, 3, 2, 1>(a, it, counter, st);
      else if (tune_far_dy())   // k2 fully unrolled: C4 far 687 -> 676 ms (x3: 687, x4: 680)
        far_packed_launch<KIND, 9, 9, 2, 2, false, true>(a, it, counter, st);
      else if (tune_far_unroll(KIND) == 3) far_packed_launch<KIND, 9, 3, 2>(a, it, counter, st);
      else far_packed_launch<KIND, 9, 1, 2>(a, it, counter, st);
      return true;
    default: return false;
  }
}

template <int KIND, int CH = kNearCh, int FORM = 0, bool PAR = false, int ABS = 0,
          bool YS = false>
void near_packed_launch(const EvalArgs& a, const PackedItems& it, int* counter,
                        cudaStream_t st) {
  const size_t smem = sizeof(double4) * kWarps * NearSmem<CH>::kWarp +
                      (YS ? sizeof(double) * (2 * kExp2WK + 1) : 0);
  auto kern = tune_near_bulk() ? k_near_packed<KIND, CH, 2, FORM, PAR, true, ABS, YS>
                               : k_near_packed<KIND, CH, 2, FORM, PAR, false, ABS, YS>;
  BLTC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = persistent_grid(kern, kWarps * 32, smem);
  kern<<<grid, kWarps * 32, smem, st>>>(a, it.items_near, it.n_items, it.poff, it.dmask,
                                        it.bys, counter);
  BLTC_LAUNCH_CHECK();
}
}  // namespace

bool packed_preferred(int kind, double chunk_lane_eff) {
  // With longest-first item order the packed kernels are at least as fast as
  // the per-batch ones at every measured batch size, including full batches
  // (N_B = 2000: C2 71.9 vs 73.3 ms, C3 169.9 vs 175.4, C4 1146 vs 1163);
  // BLTC_PACK=0 (packed_supported) still selects the per-batch kernels.
  (void)kind;
  (void)chunk_lane_eff;
  return true;
}

bool packed_supported(int kind, int degree) {
  if (const char* e = std::getenv("BLTC_PACK"))
    if (std::atoi(e) == 0) return false;
  if (kind != 0 && kind != 1) return false;
  const int m = degree + 1;
  return m >= 2 && m <= 13;   // degrees 1..12 (the paper's sweeps); others per-batch
}

namespace {
// Per item the number of lockstep steps of each kernel: far = the longest
// approximation list among its segments, near = the most direct-list
// sources among its segments (chunks of kNearCh per step), as a sort key.
__global__ void k_item_costs(int n_items, const int4* __restrict__ items, EvalArgs a,
                             uint32_t* __restrict__ cost_far, uint32_t* __restrict__ cost_near) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const int4 it = items[i];
  uint32_t mf = 0, mn = 0;
  for (int k = 0; k < it.w; ++k) {
    const int64_t b = it.z + k;
    const int32_t la = a.a_ptr[(b + 1) * a.G] - a.a_ptr[b * a.G];
    uint32_t ns = 0;
    for (int e = a.d_ptr[b * a.G]; e < a.d_ptr[(b + 1) * a.G]; ++e) {
      const EvalCluster& c = a.clusters[a.d_idx[e]];
      ns += (uint32_t)(c.stop - c.start);
    }
    mf = max(mf, (uint32_t)la);
    mn = max(mn, ns);
  }
  cost_far[i] = mf;
  // near: power-of-two cost classes, longest class first, stream order
  // within a class -- concurrently running items then read neighbouring
  // batches' (largely shared) direct-list sources while they sit in L2; an
  // exact cost order scatters them (near DRAM reads 0.85 -> 76 GB per C4
  // launch, at unchanged time)
  const uint32_t cls = mn ? min(31u, 32u - (uint32_t)__clz(mn)) : 0u;
  cost_near[i] = (cls << 27) | ((1u << 27) - 1u - (uint32_t)min(i, (1 << 27) - 1));
}

bool tune_item_sort() {
  const char* e = std::getenv("BLTC_ITEM_SORT");
  return e ? std::atoi(e) != 0 : true;
}
}  // namespace

void build_packed_items(const EvalArgs& a, PackedOrder& order, DBuf<int32_t>& pc,
                        DBuf<int32_t>& poff,
                        DBuf<int32_t>& wcnt, DBuf<int32_t>& woff, DBuf<int4>& items,
                        DBuf<uint8_t>& dmask, int64_t n_direct, DBuf<int32_t>& scan_tmp,
                        HostScratch& hs, cudaStream_t st, PackedItems* out) {
  const int64_t nb = a.nb;
  pc.resize(nb + 6);   // + 16-byte-aligned scratch: chunk slots, targets (u64)
  poff.resize(nb + 1);
  unsigned long long* cs =
      reinterpret_cast<unsigned long long*>(pc.p + ((nb + 1 + 1) & ~int64_t(1)));
  BLTC_CUDA(cudaMemsetAsync(cs, 0, 2 * sizeof(unsigned long long), st));
  k_pad_counts<<<(int)((nb + 1 + 255) / 256), 256, 0, st>>>(nb, a.bstart, a.bstop, pc.p, cs);
  BLTC_LAUNCH_CHECK();
  exclusive_scan_i32(pc.p, poff.p, nb + 1, scan_tmp, st);
  int32_t* h = (int32_t*)hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, poff.p + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaMemcpyAsync(h + 2, cs, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  const int64_t S = h[0];
  const unsigned long long* hc = reinterpret_cast<const unsigned long long*>(h + 2);
  out->chunk_lane_eff = hc[0] ? (double)hc[1] / (double)hc[0] : 1.0;
  const int64_t nw = (S + kSlots - 1) / kSlots;
  wcnt.resize(nw + 1);
  woff.resize(nw + 1);
  k_window_counts<<<(int)((nw + 1 + 255) / 256), 256, 0, st>>>(nb, poff.p, nw, wcnt.p);
  BLTC_LAUNCH_CHECK();
  exclusive_scan_i32(wcnt.p, woff.p, nw + 1, scan_tmp, st);
  BLTC_CUDA(cudaMemcpyAsync(h, woff.p + nw, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  out->n_items = h[0];
  items.resize(out->n_items + 1);
  if (nw > 0) {
    k_window_fill<<<(int)((nw + 255) / 256), 256, 0, st>>>(nb, poff.p, nw, woff.p, items.p);
    BLTC_LAUNCH_CHECK();
  }
  dmask.resize(n_direct + 1 + nb);   // entry masks, then the per-batch YS flags
  out->bys = dmask.p + n_direct + 1;
  if (nb > 0) {
    k_direct_mask<<<(int)((nb + 127) / 128), 128, 0, st>>>(nb, a.G, a.d_ptr, a.d_idx,
                                                            a.clusters, a.bcenter, a.bradius,
                                                            dmask.p, a.yk.c2, dmask.p + n_direct + 1);
    BLTC_LAUNCH_CHECK();
    if (std::getenv("BLTC_TRACE_MASK")) {   // diagnostic: share of masked entries
      std::vector<uint8_t> hm(n_direct);
      BLTC_CUDA(cudaMemcpyAsync(hm.data(), dmask.p, n_direct, cudaMemcpyDeviceToHost, st));
      BLTC_CUDA(cudaStreamSynchronize(st));
      int64_t on = 0;
      for (auto v : hm) on += v;
      std::fprintf(stderr, "[bltc] direct entries %lld, singular-mask flagged %lld\n",
                   (long long)n_direct, (long long)on);
    }
  }
  out->items = items.p;
  out->items_far = items.p;
  out->items_near = items.p;
  out->poff = poff.p;
  out->dmask = dmask.p;
  const int n = out->n_items;
  if (n > 1 && tune_item_sort()) {
    // longest-processing-time-first order for the persistent kernels' atomic
    // work counter (item order does not change any result)
    order.far.resize(n);
    order.near.resize(n);
    order.cost.resize(2 * (size_t)n);
    order.cost_sorted.resize(n);
    k_item_costs<<<(n + 255) / 256, 256, 0, st>>>(n, items.p, a, order.cost.p,
                                                  order.cost.p + n);
    BLTC_LAUNCH_CHECK();
    size_t bytes = 0;
    BLTC_CUDA(cub::DeviceRadixSort::SortPairsDescending(
        nullptr, bytes, order.cost.p, order.cost_sorted.p, items.p, order.far.p, n, 0, 32, st));
    order.tmp.resize(bytes + 1);
    BLTC_CUDA(cub::DeviceRadixSort::SortPairsDescending(order.tmp.p, bytes, order.cost.p,
                                                        order.cost_sorted.p, items.p,
                                                        order.far.p, n, 0, 32, st));
    BLTC_CUDA(cub::DeviceRadixSort::SortPairsDescending(order.tmp.p, bytes, order.cost.p + n,
                                                        order.cost_sorted.p, items.p,
                                                        order.near.p, n, 0, 32, st));
    out->items_far = order.far.p;
    out->items_near = order.near.p;
  }
}

void launch_eval_packed(const EvalArgs& a, int kind, const PackedItems& it, int* counters,
                        cudaStream_t st, float* far_ms, float* near_ms, bool timing,
                        bool parity, bool strict) {
  if (a.nb == 0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  if (timing) {
    BLTC_CUDA(cudaEventCreate(&e0));
    BLTC_CUDA(cudaEventCreate(&e1));
    BLTC_CUDA(cudaEventCreate(&e2));
  }
  BLTC_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(int), st));
  if (timing) BLTC_CUDA(cudaEventRecord(e0, st));
  if (parity) {
    if (kind == 0) far_packed_dispatch_parity<0>(a, it, counters, st);
    else far_packed_dispatch_parity<1>(a, it, counters, st);
  } else if (kind == 0) {
    far_packed_dispatch<0>(a, it, counters, st);
  } else {
    far_packed_dispatch<1>(a, it, counters, st);
  }
  if (timing) BLTC_CUDA(cudaEventRecord(e1, st));
  if (parity) {
    if (kind == 0) near_packed_launch<0, kNearCh, 0, true>(a, it, counters + 1, st);
    else near_packed_launch<1, kNearCh, 0, true>(a, it, counters + 1, st);
  } else if (strict) {   // FORM 2 arithmetic plus the |term| sums
    const int v = tune_abs();
    if (kind == 0) {
      if (v == 1) near_packed_launch<0, kNearCh, 2, false, 1>(a, it, counters + 1, st);
      else if (v == 2) near_packed_launch<0, kNearCh, 2, false, 2>(a, it, counters + 1, st);
      else near_packed_launch<0, kNearCh, 2, false, 3>(a, it, counters + 1, st);
    } else {
      if (v == 1 && tune_yshift()) near_packed_launch<1, kNearCh, 2, false, 1, true>(a, it, counters + 1, st);
      else if (v == 1) near_packed_launch<1, kNearCh, 2, false, 1>(a, it, counters + 1, st);
      else if (v == 2) near_packed_launch<1, kNearCh, 2, false, 2>(a, it, counters + 1, st);
      else near_packed_launch<1, kNearCh, 2, false, 3>(a, it, counters + 1, st);
    }
  } else if (tune_form() != 2) {
    if (kind == 0) near_packed_launch<0>(a, it, counters + 1, st);
    else near_packed_launch<1>(a, it, counters + 1, st);
  } else {
    if (kind == 0) near_packed_launch<0, kNearCh, 2>(a, it, counters + 1, st);
    else if (tune_yshift()) near_packed_launch<1, kNearCh, 2, false, 0, true>(a, it, counters + 1, st);
    else near_packed_launch<1, kNearCh, 2>(a, it, counters + 1, st);
  }
  if (timing) {
    BLTC_CUDA(cudaEventRecord(e2, st));
    BLTC_CUDA(cudaEventSynchronize(e2));
    BLTC_CUDA(cudaEventElapsedTime(far_ms, e0, e1));
    BLTC_CUDA(cudaEventElapsedTime(near_ms, e1, e2));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
  }
}

int tune_abs() {
  // measured at C4 / C3 near field: FAST 203.4 / 33.2 ms; variant 1 224.5 /
  // 35.5, 2 237.4 / 36.6, 3 224.3 / 35.2 (+14% recomputed targets): the
  // kernel is close to issue-bound, so the FP32 variants' extra integer
  // instructions cost more than one DFMA
  const char* e = std::getenv("BLTC_ABS");
  return e ? std::atoi(e) : 1;
}

}  // namespace bltc
