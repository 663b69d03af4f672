// FAST-mode evaluation: the two FP64-bound interaction kernels.
//
// far field  (_approx_tile, engine.py:216-252): batch x proxy grid
// near field (_direct_tile, engine.py:151-213): batch x cluster particles
//
// Both: one CTA per target batch (taken in descending-cost order when a work
// list is given), 128 threads, kTpt targets per thread held in registers so
// every shared-memory broadcast of a proxy / source feeds kTpt pairs.
// Reciprocal square roots use the MUFU.RSQ64H seed plus one cubic correction
// (5 FP64 ops, full double accuracy), products are fused (FMA).  Far field:
// dz^2 is hoisted per (target, k3) and dx^2 + dy^2 per (target, k1, k2), so
// the steady state is 1 DADD + rsqrt + 1 DFMA = 7 FP64 slots per pair.
// Near field: 12 slots per pair; the singular-pair test (d^2 < 1e-28,
// engine.py:175) is done on the integer pipe; per-tile partial sums are
// folded into a Neumaier-compensated per-target total (as the reference
// compensates per pair), keeping the result order-robust.
#include "bltc_internal.cuh"
#include "eval_common.cuh"

namespace bltc {

namespace {
constexpr int kThreads = 128;
constexpr int kTpt = 4;
constexpr int kPass = kThreads * kTpt;
constexpr int kSrcTile = 256;
// bit pattern of 1e-28: for d2 >= 0, (bits(d2) >= kThrBits) <=> d2 >= 1e-28
__device__ __forceinline__ long long thr_bits() { return __double_as_longlong(kSingularSq); }

__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double xy = __dmul_rn(x, y);
  const double e = fma(-xy, y, 1.0);
  const double c = fma(0.375, e, 0.5);
  const double ye = __dmul_rn(y, e);
  return fma(ye, c, y);
}

template <int KIND>
__device__ __forceinline__ double far_accum(double acc, double q, double d2, double kappa) {
  if (KIND == 0) return fma(q, rsqrt_fast(d2), acc);
  if (KIND == 1) {
    const double y = rsqrt_fast(d2);
    const double r = __dmul_rn(d2, y);
    return fma(__dmul_rn(q, exp(-kappa * r)), y, acc);
  }
  return __dadd_rn(acc, q);
}

__device__ __forceinline__ void neumaier(double& acc, double& comp, double t) {
  const double s = __dadd_rn(acc, t);
  const bool big = fabs(acc) >= fabs(t);
  const double hi = big ? acc : t, lo = big ? t : acc;
  comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(hi, s), lo));
  acc = s;
}

// ---------------------------------------------------------------------------
// Far field.  M = n + 1 known at compile time (unrolled k3); M = 0 is the
// generic runtime-degree variant.
template <int KIND, int M>
__global__ void __launch_bounds__(kThreads) k_far_fast(EvalArgs a) {
  extern __shared__ double smem[];
  const int m = M > 0 ? M : a.degree + 1;
  const int m3 = m * m * m;
  double* pts = smem;              // [3][kMaxM]
  double* qh = smem + 3 * kMaxM;   // [m3]
  const int b = a.work ? a.work[blockIdx.x] : blockIdx.x;
  const int t0 = a.bstart[b], t1 = a.bstop[b];
  const int e0 = a.a_ptr[(int64_t)b * a.G], e1 = a.a_ptr[(int64_t)(b + 1) * a.G];
  for (int pass0 = t0; pass0 < t1; pass0 += kPass) {
    double tx[kTpt], ty[kTpt], tz[kTpt], acc[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = min(pass0 + k * kThreads + (int)threadIdx.x, t1 - 1);
      tx[k] = a.tx[i];
      ty[k] = a.ty[i];
      tz[k] = a.tz[i];
      acc[k] = 0.0;
    }
    for (int e = e0; e < e1; ++e) {
      const EvalCluster c = a.clusters[a.a_idx[e]];
      __syncthreads();
      for (int i = threadIdx.x; i < 3 * m; i += kThreads) {
        const int d = i / m, k = i % m;
        pts[d * kMaxM + k] = cheb_point_dev(a.degree, k, c.lo[d], c.hi[d], a.s_nodes);
      }
      const double* row = a.moments + (size_t)c.mrow * m3;
      for (int i = threadIdx.x; i < m3; i += kThreads) qh[i] = row[i];
      __syncthreads();
      if (KIND == 2) {
        double s = 0.0;
        for (int i = 0; i < m3; ++i) s = __dadd_rn(s, qh[i]);
#pragma unroll
        for (int k = 0; k < kTpt; ++k) acc[k] = __dadd_rn(acc[k], s);
        continue;
      }
      if (M > 0) {
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
        for (int k1 = 0; k1 < M; ++k1) {
          const double p1 = pts[k1];
          double dx2[kTpt];
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const double dx = __dsub_rn(tx[k], p1);
            dx2[k] = __dmul_rn(dx, dx);
          }
          for (int k2 = 0; k2 < M; ++k2) {
            const double p2 = pts[kMaxM + k2];
            double dxy2[kTpt];
#pragma unroll
            for (int k = 0; k < kTpt; ++k) {
              const double dy = __dsub_rn(ty[k], p2);
              dxy2[k] = fma(dy, dy, dx2[k]);
            }
            const double* qr = qh + (k1 * M + k2) * M;
#pragma unroll
            for (int k3 = 0; k3 < M; ++k3) {
              const double qv = qr[k3];
#pragma unroll
              for (int k = 0; k < kTpt; ++k)
                acc[k] = far_accum<KIND>(acc[k], qv, __dadd_rn(dxy2[k], dz2[k][k3]), a.kappa);
            }
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
                acc[k] = far_accum<KIND>(acc[k], qv, fma(dz, dz, dxy2[k]), a.kappa);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = pass0 + k * kThreads + threadIdx.x;
      if (i < t1) a.far_out[i] = acc[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Near field: stream every direct cluster's sources through shared memory.
template <int KIND>
__global__ void __launch_bounds__(kThreads) k_near_fast(EvalArgs a) {
  __shared__ double4 tile[kSrcTile];
  const int b = a.work ? a.work[blockIdx.x] : blockIdx.x;
  const int t0 = a.bstart[b], t1 = a.bstop[b];
  const int e0 = a.d_ptr[(int64_t)b * a.G], e1 = a.d_ptr[(int64_t)(b + 1) * a.G];
  const long long tb = thr_bits();
  for (int pass0 = t0; pass0 < t1; pass0 += kPass) {
    double tx[kTpt], ty[kTpt], tz[kTpt], acc[kTpt], comp[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = min(pass0 + k * kThreads + (int)threadIdx.x, t1 - 1);
      tx[k] = a.tx[i];
      ty[k] = a.ty[i];
      tz[k] = a.tz[i];
      acc[k] = 0.0;
      comp[k] = 0.0;
    }
    for (int e = e0; e < e1; ++e) {
      const EvalCluster c = a.clusters[a.d_idx[e]];
      for (int j0 = c.start; j0 < c.stop; j0 += kSrcTile) {
        const int jn = min(kSrcTile, c.stop - j0);
        __syncthreads();
        for (int i = threadIdx.x; i < jn; i += kThreads) tile[i] = a.src4[j0 + i];
        __syncthreads();
        double part[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) part[k] = 0.0;
#pragma unroll 2
        for (int j = 0; j < jn; ++j) {
          const double4 s = tile[j];
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const double dx = __dsub_rn(tx[k], s.x);
            const double dy = __dsub_rn(ty[k], s.y);
            const double dz = __dsub_rn(tz[k], s.z);
            const double d2 = fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx)));
            const bool ok = __double_as_longlong(d2) >= tb;
            const double d2s = ok ? d2 : 1.0;
            const double qs = ok ? s.w : 0.0;
            if (KIND == 0) {
              part[k] = fma(qs, rsqrt_fast(d2s), part[k]);
            } else if (KIND == 1) {
              const double y = rsqrt_fast(d2s);
              const double r = __dmul_rn(d2s, y);
              part[k] = fma(__dmul_rn(qs, exp(-a.kappa * r)), y, part[k]);
            } else {
              part[k] = __dadd_rn(part[k], qs);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kTpt; ++k) neumaier(acc[k], comp[k], part[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int i = pass0 + k * kThreads + threadIdx.x;
      if (i < t1) {
        // far + near: the reference adds the approximations first, then the
        // compensated direct sums on top (engine.py:302-312, 335).
        double total = acc[k];
        double cmp = comp[k];
        neumaier(total, cmp, a.far_out[i]);
        a.out[i] = __dadd_rn(total, cmp);
      }
    }
  }
}

template <int KIND, int M>
void far_launch(const EvalArgs& a, cudaStream_t st) {
  const int m = M > 0 ? M : a.degree + 1;
  const size_t smem = sizeof(double) * (3 * kMaxM + (size_t)m * m * m);
  BLTC_CUDA(cudaFuncSetAttribute(k_far_fast<KIND, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  k_far_fast<KIND, M><<<(unsigned)a.nb, kThreads, smem, st>>>(a);
  BLTC_LAUNCH_CHECK();
}

template <int KIND>
void far_dispatch(const EvalArgs& a, cudaStream_t st) {
  switch (a.degree + 1) {
    case 5: far_launch<KIND, 5>(a, st); break;
    case 6: far_launch<KIND, 6>(a, st); break;
    case 8: far_launch<KIND, 8>(a, st); break;
    case 9: far_launch<KIND, 9>(a, st); break;
    case 11: far_launch<KIND, 11>(a, st); break;
    default: far_launch<KIND, 0>(a, st); break;
  }
}
}  // namespace

void launch_eval_fast(const EvalArgs& a, int kind, cudaStream_t st, cudaStream_t st2,
                      cudaEvent_t far_done, float* far_ms, float* near_ms, bool timing) {
  (void)st2;
  (void)far_done;
  if (a.nb == 0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  if (timing) {
    BLTC_CUDA(cudaEventCreate(&e0));
    BLTC_CUDA(cudaEventCreate(&e1));
    BLTC_CUDA(cudaEventCreate(&e2));
    BLTC_CUDA(cudaEventRecord(e0, st));
  }
  if (kind == 0) far_dispatch<0>(a, st);
  else if (kind == 1) far_dispatch<1>(a, st);
  else far_launch<2, 0>(a, st);
  if (timing) BLTC_CUDA(cudaEventRecord(e1, st));
  if (kind == 0) k_near_fast<0><<<(unsigned)a.nb, kThreads, 0, st>>>(a);
  else if (kind == 1) k_near_fast<1><<<(unsigned)a.nb, kThreads, 0, st>>>(a);
  else k_near_fast<2><<<(unsigned)a.nb, kThreads, 0, st>>>(a);
  BLTC_LAUNCH_CHECK();
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

}  // namespace bltc
