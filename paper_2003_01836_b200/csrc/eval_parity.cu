// PARITY-mode evaluation: bit-faithful to the reference tiles
// (_approx_tile engine.py:216-252, _direct_tile engine.py:151-213) driven in
// _run_batch / _eval_rank order (engine.py:296-312, decomp.py:437-454):
//   per target: for each source group: approx list (plain sum per cluster,
//   then out += acc), direct list (Neumaier into out/carry); finally
//   out + carry.
// One CTA per target batch, one thread per target (register-blocked, up to
// kTpt targets per thread and pass).  Cluster grids and moment rows, and
// direct-source tiles, are staged in shared memory and read as broadcasts.
// IEEE sqrt / division, no FMA (the library is built with -fmad=false and
// every operation here is an explicit round-to-nearest intrinsic).
#include "bltc_internal.cuh"
#include "eval_common.cuh"

namespace bltc {

namespace {
constexpr int kThreads = 256;
constexpr int kTpt = 4;
constexpr int kSrcTile = 256;

template <int KIND>
__device__ __forceinline__ double parity_term(double q, double d2, double kappa) {
  if (KIND == 0) return __ddiv_rn(q, __dsqrt_rn(d2));
  if (KIND == 1) {
    double r = __dsqrt_rn(d2);
    return __ddiv_rn(__dmul_rn(libm_exp(__dmul_rn(-kappa, r)), q), r);
  }
  return q;
}
}  // namespace

template <int KIND>
__global__ void __launch_bounds__(kThreads) k_eval_parity(EvalArgs a) {
  extern __shared__ double smem[];
  const int m = a.degree + 1;
  const int m3 = m * m * m;
  double* pts = smem;                 // [3][kMaxM]
  double* qh = smem + 3 * kMaxM;      // [m3]
  double* tile = qh + m3;             // [4][kSrcTile]
  const int b = blockIdx.x;
  const int t0 = a.bstart[b], t1 = a.bstop[b];
  for (int pass0 = t0; pass0 < t1; pass0 += kThreads * kTpt) {
    double tx[kTpt], ty[kTpt], tz[kTpt], out[kTpt], carry[kTpt];
    bool has[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      int i = pass0 + k * kThreads + threadIdx.x;
      has[k] = i < t1;
      tx[k] = has[k] ? a.tx[i] : 0.0;
      ty[k] = has[k] ? a.ty[i] : 0.0;
      tz[k] = has[k] ? a.tz[i] : 0.0;
      out[k] = 0.0;
      carry[k] = 0.0;
    }
    for (int g = 0; g < a.G; ++g) {
      const int seg = b * a.G + g;
      // ---- far field: _approx_tile per accepted cluster, list order
      for (int e = a.a_ptr[seg]; e < a.a_ptr[seg + 1]; ++e) {
        const EvalCluster c = a.clusters[a.a_idx[e]];
        __syncthreads();
        for (int i = threadIdx.x; i < 3 * m; i += kThreads) {
          int d = i / m, k = i % m;
          pts[d * kMaxM + k] = cheb_point_dev(a.degree, k, c.lo[d], c.hi[d], a.s_nodes);
        }
        const double* row = a.moments + (size_t)c.mrow * a.mstride;
        for (int i = threadIdx.x; i < m3; i += kThreads) qh[i] = row[i];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          if (!has[k]) continue;
          double acc = 0.0;
          int idx = 0;
          for (int k1 = 0; k1 < m; ++k1) {
            const double dx = __dsub_rn(tx[k], pts[k1]);
            for (int k2 = 0; k2 < m; ++k2) {
              const double dy = __dsub_rn(ty[k], pts[kMaxM + k2]);
              for (int k3 = 0; k3 < m; ++k3) {
                if (KIND == 2) {
                  acc = __dadd_rn(acc, qh[idx++]);
                  continue;
                }
                const double dz = __dsub_rn(tz[k], pts[2 * kMaxM + k3]);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                            __dmul_rn(dz, dz));
                acc = __dadd_rn(acc, parity_term<KIND>(qh[idx++], d2, a.kappa));
              }
            }
          }
          out[k] = __dadd_rn(out[k], acc);
        }
      }
      // ---- near field: _direct_tile per direct cluster, list order
      for (int e = a.d_ptr[seg]; e < a.d_ptr[seg + 1]; ++e) {
        const EvalCluster c = a.clusters[a.d_idx[e]];
        for (int j0 = c.start; j0 < c.stop; j0 += kSrcTile) {
          const int jn = min(kSrcTile, c.stop - j0);
          __syncthreads();
          for (int i = threadIdx.x; i < jn; i += kThreads) {
            tile[i] = a.sx[j0 + i];
            tile[kSrcTile + i] = a.sy[j0 + i];
            tile[2 * kSrcTile + i] = a.sz[j0 + i];
            tile[3 * kSrcTile + i] = a.sq[j0 + i];
          }
          __syncthreads();
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            if (!has[k]) continue;
            double acc = out[k], comp = carry[k];
            for (int j = 0; j < jn; ++j) {
              const double dx = __dsub_rn(tx[k], tile[j]);
              const double dy = __dsub_rn(ty[k], tile[kSrcTile + j]);
              const double dz = __dsub_rn(tz[k], tile[2 * kSrcTile + j]);
              const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                          __dmul_rn(dz, dz));
              if (d2 >= kSingularSq) {
                const double t = parity_term<KIND>(tile[3 * kSrcTile + j], d2, a.kappa);
                const double s = __dadd_rn(acc, t);
                if (fabs(acc) >= fabs(t))
                  comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(acc, s), t));
                else
                  comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(t, s), acc));
                acc = s;
              }
            }
            out[k] = acc;
            carry[k] = comp;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      int i = pass0 + k * kThreads + threadIdx.x;
      if (has[k]) a.out[i] = __dadd_rn(out[k], carry[k]);
    }
  }
}

void launch_eval_parity(const EvalArgs& a, int kind, cudaStream_t st) {
  const int m = a.degree + 1;
  size_t smem = sizeof(double) * (3 * kMaxM + (size_t)m * m * m + 4 * kSrcTile);
  if (a.nb == 0) return;
  switch (kind) {
    case 0:
      BLTC_CUDA(cudaFuncSetAttribute(k_eval_parity<0>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_eval_parity<0><<<(unsigned)a.nb, kThreads, smem, st>>>(a);
      BLTC_LAUNCH_CHECK();
      break;
    case 1:
      BLTC_CUDA(cudaFuncSetAttribute(k_eval_parity<1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_eval_parity<1><<<(unsigned)a.nb, kThreads, smem, st>>>(a);
      BLTC_LAUNCH_CHECK();
      break;
    default:
      BLTC_CUDA(cudaFuncSetAttribute(k_eval_parity<2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_eval_parity<2><<<(unsigned)a.nb, kThreads, smem, st>>>(a);
      BLTC_LAUNCH_CHECK();
      break;
  }
}

}  // namespace bltc
