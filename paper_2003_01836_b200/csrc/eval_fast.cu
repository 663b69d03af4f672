// FAST-mode evaluation: the two FP64-bound interaction kernels.
//
//   far field  (_approx_tile, engine.py:216-252): targets x (n+1)^3 proxies
//   near field (_direct_tile, engine.py:151-213): targets x cluster particles
//
// Work decomposition: a work item is (target batch, chunk of 32*kTpt
// consecutive targets).  Persistent warps pull items from a global counter,
// so batches of any size keep every lane busy and long interaction lists
// balance dynamically.  Each lane holds kTpt targets in registers; every
// proxy / source value is read once per warp from the warp's own shared-
// memory stage (filled with cp.async) and feeds kTpt pairs.
//
// Arithmetic: reciprocal square roots use the MUFU.RSQ64H seed plus one
// cubic correction (5 FP64 ops, full double accuracy); products are fused.
//   far:  dz^2 hoisted per (target, k3), dx^2 + dy^2 per (target, k1, k2):
//         steady state 1 DADD + rsqrt + 1 DFMA = 7 FP64 slots / pair
//   near: 3 DADD + 1 DMUL + 2 DFMA + rsqrt + 1 DFMA = 12 slots / pair; the
//         singular-pair test (d^2 < 1e-28, engine.py:175) runs on the integer
//         pipe; per-chunk partial sums are folded into a Neumaier-compensated
//         per-target total (the reference compensates per pair).
#include "bltc_internal.cuh"
#include "eval_common.cuh"

#include <cstdio>
#include <cstdlib>

namespace bltc {

namespace {
constexpr int kWarps = 8;               // warps per CTA
constexpr int kSrcChunk = 64;           // near-field sources per stage

__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double xy = __dmul_rn(x, y);
  const double e = fma(-xy, y, 1.0);
  const double c = fma(0.375, e, 0.5);
  const double ye = __dmul_rn(y, e);
  return fma(ye, c, y);
}

__device__ __forceinline__ void neumaier(double& acc, double& comp, double t) {
  const double s = __dadd_rn(acc, t);
  const bool big = fabs(acc) >= fabs(t);
  const double hi = big ? acc : t, lo = big ? t : acc;
  comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(hi, s), lo));
  acc = s;
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

__device__ __forceinline__ int next_item(int* counter) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, it, 0);
}


// q / sqrt(d2) accumulated into acc, full double accuracy, in the form that
// keeps 3-register-operand DFMAs (which issue at 2/3 rate on sm_100a: the
// register file delivers two 64-bit operands per cycle) to one per pair:
//   y0 = MUFU.RSQ64H(d2); e = 1 - d2 y0^2; p = 1 + e (1/2 + 3/8 e)
//   acc += (q y0) p                                  (cubic, error O(e^3))
// FORM 1 splits the last FMA into DMUL + DADD (no 3-register DFMA at all).
template <int FORM>
__device__ __forceinline__ double coulomb_acc(double acc, double q, double d2) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d2));
  const double e = fma(-__dmul_rn(d2, y0), y0, 1.0);
  const double c = fma(0.375, e, 0.5);
  const double p = fma(e, c, 1.0);
  const double qy = __dmul_rn(q, y0);
  if (FORM == 1) return __dadd_rn(acc, __dmul_rn(qy, p));
  return fma(qy, p, acc);
}

template <int KIND, int FORM>
__device__ __forceinline__ double pair_acc(double acc, double q, double d2, const YukawaK& yk) {
  if (KIND == 0) return coulomb_acc<FORM>(acc, q, d2);
  if (KIND == 1) {
    const double y = rsqrt_fast(d2);
    const double r = __dmul_rn(d2, y);
    return fma(__dmul_rn(q, exp_neg_kr(r, yk)), y, acc);
  }
  return __dadd_rn(acc, q);
}

// One (k1, k2) row of the proxy grid against kTpt targets.
template <int KIND, int M, int kTpt, int FORM>
__device__ __forceinline__ void far_row(double (&acc)[kTpt], const double* qr,
                                        const double (&dxy2)[kTpt],
                                        const double (&dz2)[kTpt][M], const YukawaK& yk) {
#pragma unroll
  for (int k3 = 0; k3 < M; ++k3) {
    const double qv = qr[k3];
#pragma unroll
    for (int k = 0; k < kTpt; ++k)
      acc[k] = pair_acc<KIND, FORM>(acc[k], qv, __dadd_rn(dxy2[k], dz2[k][k3]), yk);
  }
}

// ---------------------------------------------------------------------------
// Far field.  M = n + 1 at compile time (k3 unrolled); M = 0: runtime degree.
// One work item: targets [t0, min(t0 + 32 kTpt, t1)) of batch b against the
// batch's whole approximation list.
template <int KIND, int M, int kTpt, int FORM>
__device__ __forceinline__ void far_item(const EvalArgs& a, int b, int t0, int t1, double* pts,
                                         double* qh, int lane) {
  const int m = M > 0 ? M : a.degree + 1;
  const int m3 = m * m * m;
    double tx[kTpt], ty[kTpt], tz[kTpt], acc[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = min(t0 + k * 32 + lane, t1 - 1);
      tx[k] = a.tx[i];
      ty[k] = a.ty[i];
      tz[k] = a.tz[i];
      acc[k] = 0.0;
    }
    const int e0 = a.a_ptr[(int64_t)b * a.G], e1 = a.a_ptr[(int64_t)(b + 1) * a.G];
    for (int e = e0; e < e1; ++e) {
      const EvalCluster* c = a.clusters + a.a_idx[e];
      const double* row = a.moments + (size_t)c->mrow * a.mstride;
      __syncwarp();
      for (int i = lane; 2 * i < m3; i += 32) cp_async16(qh + 2 * i, row + 2 * i);
      cp_async_commit();
      for (int i = lane; i < 3 * m; i += 32) {
        const int d = i / m, k = i % m;
        pts[d * kMaxM + k] = cheb_point_dev(a.degree, k, c->lo[d], c->hi[d], a.s_nodes);
      }
      cp_async_wait<0>();
      __syncwarp();
      if (KIND == 2) {
        double s = 0.0;
        for (int i = 0; i < m3; ++i) s = __dadd_rn(s, qh[i]);
#pragma unroll
        for (int k = 0; k < kTpt; ++k) acc[k] = __dadd_rn(acc[k], s);
        continue;
      }
      if constexpr (M > 0) {
        double dz2[kTpt][M > 0 ? M : 1];
#pragma unroll
        for (int k3 = 0; k3 < M; ++k3) {
          const double p3 = pts[2 * kMaxM + k3];
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const double dz = __dsub_rn(tz[k], p3);
            dz2[k][k3] = __dmul_rn(dz, dz);
          }
        }
        const double* qr = qh;
        for (int k1 = 0; k1 < M; ++k1) {
          const double p1 = pts[k1];
          double dx2[kTpt];
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const double dx = __dsub_rn(tx[k], p1);
            dx2[k] = __dmul_rn(dx, dx);
          }
#pragma unroll 1
          for (int k2 = 0; k2 < M; ++k2, qr += M) {
            const double p2 = pts[kMaxM + k2];
            double dxy2[kTpt];
#pragma unroll
            for (int k = 0; k < kTpt; ++k) {
              const double dy = __dsub_rn(ty[k], p2);
              dxy2[k] = fma(dy, dy, dx2[k]);
            }
            far_row<KIND, M, kTpt, FORM>(acc, qr, dxy2, dz2, a.yk);
          }
        }
      } else {
        int idx = 0;
        for (int k1 = 0; k1 < m; ++k1) {
          const double p1 = pts[k1];
          for (int k2 = 0; k2 < m; ++k2) {
            const double p2 = pts[kMaxM + k2];
            double dxy2[kTpt];
#pragma unroll
            for (int k = 0; k < kTpt; ++k) {
              const double dx = __dsub_rn(tx[k], p1);
              const double dy = __dsub_rn(ty[k], p2);
              dxy2[k] = fma(dy, dy, __dmul_rn(dx, dx));
            }
            for (int k3 = 0; k3 < m; ++k3) {
              const double qv = qh[idx++];
              const double p3 = pts[2 * kMaxM + k3];
#pragma unroll
              for (int k = 0; k < kTpt; ++k) {
                const double dz = __dsub_rn(tz[k], p3);
                acc[k] = pair_acc<KIND, FORM>(acc[k], qv, fma(dz, dz, dxy2[k]), a.yk);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = t0 + k * 32 + lane;
      if (i < t1) a.far_out[i] = acc[k];
    }
}

template <int KIND, int M, int kTpt, int MINB, int FORM>
__global__ void __launch_bounds__(kWarps * 32, MINB)
k_far_fast(EvalArgs a, const int2* __restrict__ items, int n_items, int* counter) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = 3 * kMaxM + 1 + a.mstride;   // +1 keeps qh 16-byte aligned
  double* pts = smem + warp * per_warp;   // [3][kMaxM]
  double* qh = pts + 3 * kMaxM + 1;       // [mstride]
  for (int item = next_item(counter); item < n_items; item = next_item(counter)) {
    const int2 it = items[item];
    const int t1 = a.bstop[it.x];
    // a batch's last chunk with <= 32 targets runs one target per lane
    if (kTpt > 1 && t1 - it.y <= 32)
      far_item<KIND, M, 1, FORM>(a, it.x, it.y, t1, pts, qh, lane);
    else
      far_item<KIND, M, kTpt, FORM>(a, it.x, it.y, t1, pts, qh, lane);
  }
}

// ---------------------------------------------------------------------------
// Near field: each direct cluster's sources stream through a double-buffered
// per-warp stage of kSrcChunk packed (x, y, z, q) records.
__device__ __forceinline__ void stage_sources(double4* dst, const double4* src, int base,
                                              int stop, int lane) {
  for (int jj = lane; jj < kSrcChunk; jj += 32) {
    const int js = base + jj;
    if (js < stop) {
      cp_async16(&dst[jj], &src[js]);
      cp_async16(reinterpret_cast<char*>(&dst[jj]) + 16,
                 reinterpret_cast<const char*>(&src[js]) + 16);
    }
  }
  cp_async_commit();
}

// Lower bound on the distance between the batch's bounding ball and a
// cluster box (0 when they overlap).
__device__ __forceinline__ double ball_box_gap(const double* bc, double br, const EvalCluster& c) {
  double g2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double lo = c.lo[d] - bc[d], hi = bc[d] - c.hi[d];
    const double g = fmax(fmax(lo, hi), 0.0);
    g2 = fma(g, g, g2);
  }
  return sqrt(g2) - br;
}

// One staged chunk of sources against kTpt targets.  MASKED applies the
// reference's singular-pair exclusion (d^2 < 1e-28 skipped, engine.py:175)
// on the integer pipe; the unmasked variant is used when no pair can be
// singular.
template <int KIND, int kTpt, int FORM, bool MASKED>
__device__ __forceinline__ void near_chunk(double (&part)[kTpt], const double4* src, int jn,
                                           const double (&tx)[kTpt], const double (&ty)[kTpt],
                                           const double (&tz)[kTpt], const YukawaK& yk) {
  const long long tb = __double_as_longlong(kSingularSq);   // d2 >= 0: bit order = value order
#pragma unroll 4
  for (int j = 0; j < jn; ++j) {
    const double4 s = src[j];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const double dx = __dsub_rn(tx[k], s.x);
      const double dy = __dsub_rn(ty[k], s.y);
      const double dz = __dsub_rn(tz[k], s.z);
      if (MASKED) {
        // d2 + 1e-300: exactly d2 for every non-singular pair, never 0, so
        // only the charge needs the select (excluded pairs add 0 * finite)
        const double d2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, 1e-300)));
        const bool ok = __double_as_longlong(d2) >= tb;
        part[k] = pair_acc<KIND, FORM>(part[k], ok ? s.w : 0.0, d2, yk);
      } else {
        const double d2 = fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx)));
        part[k] = pair_acc<KIND, FORM>(part[k], s.w, d2, yk);
      }
    }
  }
}

template <int KIND, int kTpt, int FORM>
__device__ __forceinline__ void near_item(const EvalArgs& a, int b, int t0, int t1,
                                          double4 (*stage)[kSrcChunk], int lane) {
    double tx[kTpt], ty[kTpt], tz[kTpt], acc[kTpt], comp[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = min(t0 + k * 32 + lane, t1 - 1);
      tx[k] = a.tx[i];
      ty[k] = a.ty[i];
      tz[k] = a.tz[i];
      acc[k] = 0.0;
      comp[k] = 0.0;
    }
    const int e0 = a.d_ptr[(int64_t)b * a.G], e1 = a.d_ptr[(int64_t)(b + 1) * a.G];
    for (int e = e0; e < e1; ++e) {
      const EvalCluster c = a.clusters[a.d_idx[e]];
      const int nchunks = (c.stop - c.start + kSrcChunk - 1) / kSrcChunk;
      // The singular-pair test can only fire if the batch ball comes within
      // ~1e-14 of the cluster box; otherwise the unmasked loop is exact.
      const double* bc = a.bcenter + 3 * b;
      const double scale =
          fmax(fmax(fabs(bc[0]), fabs(bc[1])), fabs(bc[2])) + a.bradius[b];
      const bool masked = ball_box_gap(bc, a.bradius[b], c) <= 1e-12 * (1.0 + scale);
      __syncwarp();
      stage_sources(stage[0], a.src4, c.start, c.stop, lane);
      for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nchunks) {
          stage_sources(stage[buf ^ 1], a.src4, c.start + (ch + 1) * kSrcChunk, c.stop,
                        lane);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        const int jn = min(kSrcChunk, c.stop - (c.start + ch * kSrcChunk));
        double part[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) part[k] = 0.0;
        if (masked)
          near_chunk<KIND, kTpt, FORM, true>(part, stage[buf], jn, tx, ty, tz, a.yk);
        else
          near_chunk<KIND, kTpt, FORM, false>(part, stage[buf], jn, tx, ty, tz, a.yk);
#pragma unroll
        for (int k = 0; k < kTpt; ++k) neumaier(acc[k], comp[k], part[k]);
        __syncwarp();
      }
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = t0 + k * 32 + lane;
      if (i < t1) {
        // approximations first, then the compensated direct sums on top
        // (engine.py:302-312, 335)
        double total = acc[k], cmp = comp[k];
        neumaier(total, cmp, a.far_out[i]);
        a.out[i] = __dadd_rn(total, cmp);
      }
    }
}

template <int KIND, int kTpt, int MINB, int FORM>
__global__ void __launch_bounds__(kWarps * 32, MINB)
k_near_fast(EvalArgs a, const int2* __restrict__ items, int n_items, int* counter) {
  __shared__ __align__(16) double4 stage[kWarps][2][kSrcChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int item = next_item(counter); item < n_items; item = next_item(counter)) {
    const int2 it = items[item];
    const int t1 = a.bstop[it.x];
    if (kTpt > 1 && t1 - it.y <= 32)
      near_item<KIND, 1, FORM>(a, it.x, it.y, t1, stage[warp], lane);
    else
      near_item<KIND, kTpt, FORM>(a, it.x, it.y, t1, stage[warp], lane);
  }
}

__global__ void k_count_chunks(int64_t nb, const int32_t* bstart, const int32_t* bstop,
                               int kChunkT, int32_t* cnt) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < nb) cnt[b] = (bstop[b] - bstart[b] + kChunkT - 1) / kChunkT;
  if (b == nb) cnt[b] = 0;
}

__global__ void k_fill_items(int64_t nb, const int32_t* bstart, const int32_t* cnt,
                             const int32_t* off, int kChunkT, int2* items) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  for (int k = 0; k < cnt[b]; ++k) items[off[b] + k] = make_int2((int)b, bstart[b] + k * kChunkT);
}

template <typename K>
int persistent_grid(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  BLTC_CUDA(cudaGetDevice(&dev));
  BLTC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  BLTC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  return sms * (per_sm > 0 ? per_sm : 1);
}

template <int KIND, int M, int TPT, int MINB, int FORM = 0>
void far_launch(const EvalArgs& a, const FastItems& it, int* counter, cudaStream_t st) {
  const size_t smem = sizeof(double) * kWarps * (3 * kMaxM + 1 + (size_t)a.mstride);
  auto kern = k_far_fast<KIND, M, TPT, MINB, FORM>;
  BLTC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = persistent_grid(kern, kWarps * 32, smem);
  kern<<<grid, kWarps * 32, smem, st>>>(a, it.items, it.n_items, counter);
  BLTC_LAUNCH_CHECK();
}

// Tuned variants exist for the benchmark shape (Coulomb, n = 8); every other
// (kernel, degree) uses (kTpt, minBlocks) = (2, 2).
template <int KIND, int M>
void far_variant(const EvalArgs& a, const FastItems& it, int* counter, cudaStream_t st,
                 const FastTuning& t) {
  if (KIND == 0 && M == 9) {
    if (t.far_tpt == 1 && t.far_minb == 4) return far_launch<KIND, M, 1, 4>(a, it, counter, st);
    if (t.far_tpt == 2 && t.far_minb == 3) return far_launch<KIND, M, 2, 3>(a, it, counter, st);
    if (t.far_tpt == 4 && t.far_minb == 2) return far_launch<KIND, M, 4, 2>(a, it, counter, st);
    if (t.far_tpt == 3 && t.far_minb == 2) return far_launch<KIND, M, 3, 2>(a, it, counter, st);
    if (t.far_tpt == 2 && t.far_minb == 2 && t.form == 1)
      return far_launch<KIND, M, 2, 2, 1>(a, it, counter, st);
  }
  far_launch<KIND, M, 2, 2>(a, it, counter, st);
}

template <int KIND>
void far_dispatch(const EvalArgs& a, const FastItems& it, int* counter, cudaStream_t st,
                  const FastTuning& t) {
  switch (a.degree + 1) {
    case 5: far_variant<KIND, 5>(a, it, counter, st, t); break;
    case 6: far_variant<KIND, 6>(a, it, counter, st, t); break;
    case 8: far_variant<KIND, 8>(a, it, counter, st, t); break;
    case 9: far_variant<KIND, 9>(a, it, counter, st, t); break;
    case 11: far_variant<KIND, 11>(a, it, counter, st, t); break;
    default: far_launch<KIND, 0, 2, 2>(a, it, counter, st); break;
  }
}

template <int KIND, int TPT, int MINB, int FORM = 0>
void near_launch(const EvalArgs& a, const FastItems& it, int* counter, cudaStream_t st) {
  auto kern = k_near_fast<KIND, TPT, MINB, FORM>;
  const int grid = persistent_grid(kern, kWarps * 32, 0);
  kern<<<grid, kWarps * 32, 0, st>>>(a, it.items, it.n_items, counter);
  BLTC_LAUNCH_CHECK();
}

template <int KIND>
void near_variant(const EvalArgs& a, const FastItems& it, int* counter, cudaStream_t st,
                  const FastTuning& t) {
  if (KIND == 0) {
    if (t.near_tpt == 1 && t.near_minb == 4) return near_launch<KIND, 1, 4>(a, it, counter, st);
    if (t.near_tpt == 2 && t.near_minb == 3) return near_launch<KIND, 2, 3>(a, it, counter, st);
    if (t.near_tpt == 2 && t.near_minb == 4) return near_launch<KIND, 2, 4>(a, it, counter, st);
    if (t.near_tpt == 4 && t.near_minb == 2) return near_launch<KIND, 4, 2>(a, it, counter, st);
    if (t.near_tpt == 2 && t.near_minb == 2 && t.form == 1)
      return near_launch<KIND, 2, 2, 1>(a, it, counter, st);
  }
  near_launch<KIND, 2, 2>(a, it, counter, st);
}
}  // namespace

FastTuning fast_tuning() {
  FastTuning t{2, 2, 2, 2, 0};
  if (const char* e = std::getenv("BLTC_FORM")) t.form = std::atoi(e);
  if (const char* e = std::getenv("BLTC_FAR")) std::sscanf(e, "%d,%d", &t.far_tpt, &t.far_minb);
  if (const char* e = std::getenv("BLTC_NEAR"))
    std::sscanf(e, "%d,%d", &t.near_tpt, &t.near_minb);
  return t;
}

void build_fast_items(const EvalArgs& a, int chunk, DBuf<int32_t>& cnt, DBuf<int32_t>& off,
                      DBuf<int2>& items, DBuf<int32_t>& scan_tmp, HostScratch& hs,
                      cudaStream_t st, FastItems* out) {
  const int64_t nb = a.nb;
  cnt.resize(nb + 1);
  off.resize(nb + 1);
  k_count_chunks<<<(int)((nb + 1 + 255) / 256), 256, 0, st>>>(nb, a.bstart, a.bstop, chunk,
                                                               cnt.p);
  BLTC_LAUNCH_CHECK();
  exclusive_scan_i32(cnt.p, off.p, nb + 1, scan_tmp, st);
  int32_t* h = (int32_t*)hs.get(64);
  BLTC_CUDA(cudaMemcpyAsync(h, off.p + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  BLTC_CUDA(cudaStreamSynchronize(st));
  out->n_items = h[0];
  items.resize(out->n_items + 1);
  k_fill_items<<<(int)((nb + 255) / 256), 256, 0, st>>>(nb, a.bstart, cnt.p, off.p, chunk,
                                                        items.p);
  BLTC_LAUNCH_CHECK();
  out->items = items.p;
  out->chunk = chunk;
}

void launch_eval_fast(const EvalArgs& a, int kind, const FastItems& far_items,
                      const FastItems& near_items, const FastTuning& t, int* counters,
                      cudaStream_t st, float* far_ms, float* near_ms, bool timing) {
  if (a.nb == 0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  if (timing) {
    BLTC_CUDA(cudaEventCreate(&e0));
    BLTC_CUDA(cudaEventCreate(&e1));
    BLTC_CUDA(cudaEventCreate(&e2));
  }
  BLTC_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(int), st));
  if (timing) BLTC_CUDA(cudaEventRecord(e0, st));
  if (kind == 0) far_dispatch<0>(a, far_items, counters, st, t);
  else if (kind == 1) far_dispatch<1>(a, far_items, counters, st, t);
  else far_launch<2, 0, 2, 2>(a, far_items, counters, st);
  if (timing) BLTC_CUDA(cudaEventRecord(e1, st));
  if (kind == 0) near_variant<0>(a, near_items, counters + 1, st, t);
  else if (kind == 1) near_launch<1, 2, 2>(a, near_items, counters + 1, st);
  else near_launch<2, 2, 2>(a, near_items, counters + 1, st);
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

// Whether the per-batch FAST far kernel's shared-memory slab (a whole
// moment row per warp) fits the device's opt-in limit: up to degree 14.
bool fast_far_fits(int degree) {
  const int m = degree + 1;
  const int m3 = m * m * m;
  const size_t smem = sizeof(double) * kWarps * (3 * kMaxM + 1 + (size_t)((m3 + 1) & ~1));
  int dev = 0, limit = 0;
  BLTC_CUDA(cudaGetDevice(&dev));
  BLTC_CUDA(cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return smem <= (size_t)limit;
}

}  // namespace bltc
