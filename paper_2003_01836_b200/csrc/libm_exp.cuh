// Bitwise port of the host exp the reference's Yukawa tiles call.
//
// numba lowers `math.exp` in _direct_tile / _approx_tile (engine.py:190-191,
// 243) to llvm.exp.f64, i.e. a call to the process's C library exp: glibc
// 2.39's __exp (sysdeps/ieee754/dbl-64/e_exp.c, the table-driven algorithm
// with N = 2^7 and a degree-5 polynomial).  On x86-64 hosts with FMA (the
// build container and the GPU boxes) the ifunc selects the variant compiled
// with -mfma, whose contractions are read off its machine code (libm.so.6,
// the fma clone of __exp):
//   kd  = fma(x, InvLn2N, Shift)              ki = bits(kd);  kd -= Shift
//   r   = fma(kd, NegLn2loN, fma(kd, NegLn2hiN, x))
//   tmp = fma(r2 * r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, tail + r))
//   exp = fma(scale, tmp, scale)
// and the special cases (tiny |x| -> 1 + x, |x| >= 512 through specialcase
// with an unfused scale * tmp, |x| >= 1024 -> 0 / inf / NaN) likewise.
// The 2^(k/128) table is generated from first principles
// (tools/gen_exp_table.py); tests/test_libm_exp.py checks the table against
// libm's and this function against libm's exp bit for bit on the host, and
// tests/test_gpu_parity.py the device build against the host's.
#pragma once
#include <cstdint>
#include <cstring>

#include "libm_exp_table.h"

#if defined(__CUDACC__)
#define BLTC_HD __host__ __device__ __forceinline__
#else
#define BLTC_HD inline
#endif

namespace bltc {

#if defined(__CUDACC__)
static __device__ const uint64_t kExpTabDev[256] = BLTC_EXP_TABLE_INIT;
#endif
static const uint64_t kExpTabHost[256] = BLTC_EXP_TABLE_INIT;

namespace libm_detail {
BLTC_HD uint64_t as_u64(double v) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(v);
#else
  uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
#endif
}
BLTC_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double v;
  std::memcpy(&v, &u, 8);
  return v;
#endif
}
// IEEE round-to-nearest operations that no compiler may contract or reorder
BLTC_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double s = a + b;
  return s;
#endif
}
BLTC_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  volatile double s = a - b;
  return s;
#endif
}
BLTC_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double s = a * b;
  return s;
#endif
}
BLTC_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}
BLTC_HD uint64_t tab(int i) {
#if defined(__CUDA_ARCH__)
  return __ldg(reinterpret_cast<const unsigned long long*>(kExpTabDev) + i);
#else
  return kExpTabHost[i];
#endif
}
}  // namespace libm_detail

// exp(x), bitwise glibc 2.39 x86-64 (fma variant), for every double x
// (the errno / floating-point-flag side effects are not modelled).
BLTC_HD double libm_exp(double x) {
  using namespace libm_detail;
  const double kInvLn2N = 0x1.71547652b82fep0 * 128;
  const double kShift = 0x1.8p52;
  const double kNegLn2hiN = -0x1.62e42fefa0000p-8;
  const double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double kC2 = 0x1.ffffffffffdbdp-2;
  const double kC3 = 0x1.555555555543cp-3;
  const double kC4 = 0x1.55555cf172b91p-5;
  const double kC5 = 0x1.1111167a4d017p-7;
  const uint64_t ux = as_u64(x);
  uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return add(x, 1.0);   // |x| < 2^-54
    if (abstop > 0x408u) {                                     // |x| >= 1024
      if (ux == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return add(x, 1.0);
      if (ux >> 63) return 0.0;                                // underflow
      return as_f64(0x7ff0000000000000ull);                    // overflow
    }
    abstop = 0;   // 512 <= |x| < 1024: specialcase below
  }
  double kd = fma_(x, kInvLn2N, kShift);
  const uint64_t ki = as_u64(kd);
  kd = sub(kd, kShift);
  const double r = fma_(kd, kNegLn2loN, fma_(kd, kNegLn2hiN, x));
  const int idx = 2 * (int)(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = as_f64(tab(idx));
  uint64_t sbits = tab(idx + 1) + top;
  const double p1 = fma_(r, kC3, kC2);
  const double t0 = add(r, tail);
  const double r2 = mul(r, r);
  const double p2 = fma_(r, kC5, kC4);
  const double t1 = fma_(p1, r2, t0);
  const double r4 = mul(r2, r2);
  const double tmp = fma_(r4, p2, t1);
  if (abstop != 0) {
    const double scale = as_f64(sbits);
    return fma_(scale, tmp, scale);
  }
  if ((ki & 0x80000000u) == 0) {   // k > 0: scale's exponent may overflow
    sbits -= 1009ull << 52;
    const double scale = as_f64(sbits);
    return mul(fma_(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;          // k < 0: subnormal range
  const double scale = as_f64(sbits);
  const double st = mul(tmp, scale);
  double y = add(scale, st);
  if (1.0 > y) {
    const double hi = add(y, 1.0);
    const double lo = add(sub(scale, y), st);
    double v = add(sub(1.0, hi), y);
    v = add(v, lo);
    v = add(v, hi);
    y = sub(v, 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul(y, 0x1p-1022);
}

}  // namespace bltc
