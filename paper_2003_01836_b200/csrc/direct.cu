// Brute-force direct sums at (sampled) targets over all sources -- the
// verification oracle of the reference harness (cli.py:73-149,
// _oracle_kernel) on the GPU, so full-N errors at 1M-64M
// take seconds instead of CPU hours.
//
// PARITY: one thread per target, sources in ascending order, IEEE sqrt/div,
// Neumaier compensation -- bitwise the CPU oracle for Coulomb / constant.
// FAST: sources split into kSplit pieces, each (64-target, piece) work item
// accumulates rsqrt-based terms with per-chunk Neumaier folding; pieces are
// combined per target in piece order (deterministic).
#include "bltc_internal.cuh"
#include "eval_common.cuh"

namespace bltc {

namespace {
constexpr int kThreads = 128;
constexpr int kTile = 256;
constexpr int kSplit = 1 << 16;

template <int KIND>
__device__ __forceinline__ double ieee_term(double q, double d2, double kappa) {
  if (KIND == 0) return __ddiv_rn(q, __dsqrt_rn(d2));
  if (KIND == 1) {
    const double r = __dsqrt_rn(d2);
    return __ddiv_rn(__dmul_rn(libm_exp(__dmul_rn(-kappa, r)), q), r);
  }
  return q;
}

__device__ __forceinline__ void neumaier_add(double& acc, double& comp, double t) {
  const double s = __dadd_rn(acc, t);
  if (fabs(acc) >= fabs(t))
    comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(acc, s), t));
  else
    comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(t, s), acc));
  acc = s;
}

__device__ __forceinline__ double rsqrt_f(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-__dmul_rn(x, y), y, 1.0);
  return __dmul_rn(y, fma(e, fma(0.375, e, 0.5), 1.0));
}

template <int KIND>
__global__ void __launch_bounds__(kThreads)
k_direct_parity(int64_t n_idx, const int64_t* __restrict__ idx, const double* __restrict__ tx,
                const double* __restrict__ ty, const double* __restrict__ tz, int64_t ns,
                const double* __restrict__ sx, const double* __restrict__ sy,
                const double* __restrict__ sz, const double* __restrict__ sq, double kappa,
                double* __restrict__ out) {
  __shared__ double tile[4][kTile];
  const int64_t a = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const bool has = a < n_idx;
  const int64_t i = has ? idx[a] : 0;
  const double xi = tx[i], yi = ty[i], zi = tz[i];
  double acc = 0.0, comp = 0.0;
  for (int64_t j0 = 0; j0 < ns; j0 += kTile) {
    const int jn = (int)(ns - j0 < kTile ? ns - j0 : kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jn; j += kThreads) {
      tile[0][j] = sx[j0 + j];
      tile[1][j] = sy[j0 + j];
      tile[2][j] = sz[j0 + j];
      tile[3][j] = sq[j0 + j];
    }
    __syncthreads();
    for (int j = 0; j < jn; ++j) {
      const double dx = __dsub_rn(xi, tile[0][j]);
      const double dy = __dsub_rn(yi, tile[1][j]);
      const double dz = __dsub_rn(zi, tile[2][j]);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (d2 >= kSingularSq) neumaier_add(acc, comp, ieee_term<KIND>(tile[3][j], d2, kappa));
    }
  }
  if (has) out[a] = __dadd_rn(acc, comp);
}

// FAST: item (target block, source piece); partial (acc, comp) per target.
template <int KIND>
__global__ void __launch_bounds__(kThreads)
k_direct_fast(int64_t n_idx, const int64_t* __restrict__ idx, const double* __restrict__ tx,
              const double* __restrict__ ty, const double* __restrict__ tz, int64_t ns,
              const double4* __restrict__ src, double kappa, double2* __restrict__ partial) {
  __shared__ double4 tile[kTile];
  const int64_t a = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const int piece = blockIdx.y;
  const bool has = a < n_idx;
  const int64_t i = has ? idx[a] : 0;
  const double xi = tx[i], yi = ty[i], zi = tz[i];
  const long long tb = __double_as_longlong(kSingularSq);
  double acc = 0.0, comp = 0.0;
  const int64_t p0 = (int64_t)piece * kSplit;
  const int64_t p1 = (ns < p0 + kSplit ? ns : p0 + kSplit);
  for (int64_t j0 = p0; j0 < p1; j0 += kTile) {
    const int jn = (int)(p1 - j0 < kTile ? p1 - j0 : kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jn; j += kThreads) tile[j] = src[j0 + j];
    __syncthreads();
    double part = 0.0;
#pragma unroll 4
    for (int j = 0; j < jn; ++j) {
      const double4 s = tile[j];
      const double dx = __dsub_rn(xi, s.x);
      const double dy = __dsub_rn(yi, s.y);
      const double dz = __dsub_rn(zi, s.z);
      const double d2 = fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx)));
      const bool ok = __double_as_longlong(d2) >= tb;
      const double d2s = ok ? d2 : 1.0, qs = ok ? s.w : 0.0;
      if (KIND == 0) {
        part = fma(qs, rsqrt_f(d2s), part);
      } else if (KIND == 1) {
        const double y = rsqrt_f(d2s);
        part = fma(__dmul_rn(qs, exp(-kappa * __dmul_rn(d2s, y))), y, part);
      } else {
        part = __dadd_rn(part, qs);
      }
    }
    neumaier_add(acc, comp, part);
  }
  if (has) partial[(int64_t)piece * n_idx + a] = make_double2(acc, comp);
}

__global__ void k_direct_reduce(int64_t n_idx, int pieces, const double2* __restrict__ partial,
                                double* __restrict__ out) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n_idx) return;
  double acc = 0.0, comp = 0.0;
  for (int p = 0; p < pieces; ++p) {
    const double2 v = partial[(int64_t)p * n_idx + a];
    neumaier_add(acc, comp, v.x);
    comp = __dadd_rn(comp, v.y);
  }
  out[a] = __dadd_rn(acc, comp);
}

__global__ void k_pack_sources(int64_t n, const double* x, const double* y, const double* z,
                               const double* q, double4* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double4(x[i], y[i], z[i], q[i]);
}
}  // namespace

void direct_sum_device(int kind, double kappa, int mode, int64_t n_idx, const int64_t* idx,
                       const double* tx, const double* ty, const double* tz, int64_t ns,
                       const double* sx, const double* sy, const double* sz, const double* sq,
                       double* out, DBuf<double4>& src4, DBuf<double2>& partial,
                       cudaStream_t st) {
  if (n_idx <= 0) return;
  const unsigned nb = (unsigned)((n_idx + kThreads - 1) / kThreads);
  if (mode == BLTC_MODE_PARITY) {
    if (kind == 0)
      k_direct_parity<0><<<nb, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, sx, sy, sz, sq,
                                                  kappa, out);
    else if (kind == 1)
      k_direct_parity<1><<<nb, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, sx, sy, sz, sq,
                                                  kappa, out);
    else
      k_direct_parity<2><<<nb, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, sx, sy, sz, sq,
                                                  kappa, out);
    BLTC_LAUNCH_CHECK();
    return;
  }
  src4.resize(ns);
  k_pack_sources<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(ns, sx, sy, sz, sq, src4.p);
  BLTC_LAUNCH_CHECK();
  const int pieces = (int)((ns + kSplit - 1) / kSplit);
  partial.resize((size_t)pieces * n_idx);
  dim3 grid(nb, pieces);
  if (kind == 0)
    k_direct_fast<0><<<grid, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, src4.p, kappa,
                                                partial.p);
  else if (kind == 1)
    k_direct_fast<1><<<grid, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, src4.p, kappa,
                                                partial.p);
  else
    k_direct_fast<2><<<grid, kThreads, 0, st>>>(n_idx, idx, tx, ty, tz, ns, src4.p, kappa,
                                                partial.p);
  BLTC_LAUNCH_CHECK();
  k_direct_reduce<<<nb, kThreads, 0, st>>>(n_idx, pieces, partial.p, out);
  BLTC_LAUNCH_CHECK();
}

}  // namespace bltc
