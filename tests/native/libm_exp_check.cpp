// Host check of bltc::libm_exp (csrc/libm_exp.cuh) against the C library's
// exp, bit for bit: argv[1] random samples per range, argv[2] seed.
// Prints "mismatches <n> checked <m>" and the first few mismatches.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "libm_exp.cuh"

static double (*volatile host_exp)(double) = std::exp;

static uint64_t bits(double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
  const unsigned seed = argc > 2 ? (unsigned)std::atoi(argv[2]) : 1u;
  std::mt19937_64 rng(seed);
  long bad = 0, checked = 0;
  auto check = [&](double x) {
    const double a = bltc::libm_exp(x), b = host_exp(x);
    ++checked;
    if (bits(a) != bits(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 8) std::printf("x=%a port=%a libm=%a\n", x, a, b);
      ++bad;
    }
  };
  const double specials[] = {0.0, -0.0, 1e-300, -1e-300, 0x1p-54, -0x1p-54, 0x1p-55, -0x1p-53,
                             1.0, -1.0, 512.0, -512.0, 709.7, 709.8, -708.4, -745.1, -745.2,
                             -1024.0, 1024.0, -1e300, 1e300, INFINITY, -INFINITY, NAN,
                             4.9e-324, -4.9e-324, -0.5, -3.5, -0x1.62e42fefa39efp-1};
  for (double s : specials) check(s);
  std::uniform_real_distribution<double> wide(-1100.0, 1100.0), neg(-20.0, 0.0),
      unit(0.0, 1.0), expo(-60.0, 11.0);
  for (long i = 0; i < n; ++i) {
    check(wide(rng));
    check(neg(rng));
    // Yukawa arguments: -kappa * r, r = sqrt(d2)
    const double kappa = i % 3 == 0 ? 0.5 : (i % 3 == 1 ? 1.0 : 7.25);
    check(-kappa * std::sqrt(3.0 * unit(rng) * unit(rng)));
    const double m = std::ldexp(1.0 + unit(rng), (int)expo(rng));
    check(i & 1 ? -m : m);
    uint64_t u = rng();   // arbitrary bit patterns
    double v;
    std::memcpy(&v, &u, 8);
    check(v);
  }
  std::printf("mismatches %ld checked %ld\n", bad, checked);
  return bad != 0;
}
