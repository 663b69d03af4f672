/* libbltc from plain C: no Python, no torch -- the drop-in boundary as a
 * maintainer of any host language would bind it (include/bltc.h).
 *
 *   gcc -O2 -Iinclude examples/treecode_c.c -o treecode_c \
 *       -Lpaper_2003_01836_b200 -lbltc -Wl,-rpath,$PWD/paper_2003_01836_b200 -lm
 *   ./treecode_c [n]
 *
 * Uniform random particles in [-1,1]^3 (an LCG, not the harness's Philox
 * stream), Coulomb, n = 6, theta = 0.7: the treecode potentials in PARITY
 * and FAST mode, checked against a brute-force direct sum on a sample of
 * targets (relative L2 error, cli.py:152-159) and against each other; then
 * a 2-rank bltc_run_distributed over a median split in x (any partition the
 * caller chooses; decomp.rcb_partition's is the reference's). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bltc.h"

static const double* sort_key;
static int by_key(const void* a, const void* b) {
  const double u = sort_key[*(const int64_t*)a], v = sort_key[*(const int64_t*)b];
  return (u > v) - (u < v);
}

static uint64_t lcg = 0x9E3779B97F4A7C15ull;
static double uniform(void) {
  lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
  return -1.0 + 2.0 * (double)(lcg >> 11) * (1.0 / 9007199254740992.0);
}

#define CHECK(call)                                                             \
  do {                                                                          \
    int rc_ = (call);                                                           \
    if (rc_ != BLTC_OK) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, bltc_last_error());   \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 50000;
  double *x = malloc(n * sizeof(double)), *y = malloc(n * sizeof(double));
  double *z = malloc(n * sizeof(double)), *q = malloc(n * sizeof(double));
  double *phi_p = malloc(n * sizeof(double)), *phi_f = malloc(n * sizeof(double));
  double* phi_s = malloc(n * sizeof(double));
  double* phi_d = malloc(n * sizeof(double));
  int64_t* order = malloc(n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    x[i] = uniform();
    y[i] = uniform();
    z[i] = uniform();
    q[i] = uniform();
  }
  const int degree = 6;
  double s[7];   /* Chebyshev nodes sin(pi (n - 2k) / (2n)) (interp.py:35-56) */
  for (int k = 0; k <= degree; ++k) s[k] = sin(3.141592653589793 * (degree - 2 * k) / (2.0 * degree));
  bltc_params p = {0.7, degree, 0, 500, 500, 0.0, BLTC_MODE_PARITY, 0};
  bltc_ctx* ctx = NULL;
  bltc_stats st;
  CHECK(bltc_create(0, NULL, &ctx));
  CHECK(bltc_treecode(ctx, &p, s, n, x, y, z, n, x, y, z, q, 1, phi_p, &st));
  p.mode = BLTC_MODE_STRICT;   /* the default of the Python shim */
  CHECK(bltc_treecode(ctx, &p, s, n, x, y, z, n, x, y, z, q, 1, phi_s, &st));
  p.mode = BLTC_MODE_FAST;
  CHECK(bltc_treecode(ctx, &p, s, n, x, y, z, n, x, y, z, q, 1, phi_f, &st));
  /* a bad parameter is reported, not thrown */
  bltc_params bad = p;
  bad.theta = 1.5;
  if (bltc_treecode(ctx, &bad, s, n, x, y, z, n, x, y, z, q, 1, phi_f, NULL) != BLTC_ERR_VALUE) {
    fprintf(stderr, "theta = 1.5 was not rejected\n");
    return 1;
  }
  CHECK(bltc_destroy(ctx));
  /* two ranks: lower / upper half in x, both on device 0 */
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  sort_key = x;
  qsort(order, (size_t)n, sizeof(int64_t), by_key);
  const int64_t rank_start[3] = {0, n / 2, n};
  const int32_t devices[1] = {0};
  bltc_stats dst;
  CHECK(bltc_run_distributed(2, devices, 1, &p, s, n, x, y, z, q, order, rank_start, phi_d,
                             &dst));
  /* direct sum on every 97th target, Neumaier-compensated */
  double num = 0.0, den = 0.0, numd = 0.0, dev = 0.0, scale = 0.0;
  for (int64_t i = 0; i < n; i += 97) {
    double acc = 0.0, comp = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double dx = x[i] - x[j], dy = y[i] - y[j], dz = z[i] - z[j];
      const double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 < 1e-28) continue;
      const double t = q[j] / sqrt(d2), sum = acc + t;
      comp += fabs(acc) >= fabs(t) ? (acc - sum) + t : (t - sum) + acc;
      acc = sum;
    }
    const double ds = acc + comp;
    num += (phi_p[i] - ds) * (phi_p[i] - ds);
    numd += (phi_d[i] - ds) * (phi_d[i] - ds);
    den += ds * ds;
  }
  double strict = 0.0;   /* STRICT: per target, against PARITY (= the reference) */
  for (int64_t i = 0; i < n; ++i) {
    dev = fmax(dev, fabs(phi_f[i] - phi_p[i]));
    scale = fmax(scale, fabs(phi_p[i]));
    if (phi_p[i] != 0.0) strict = fmax(strict, fabs(phi_s[i] - phi_p[i]) / fabs(phi_p[i]));
  }
  const double err = sqrt(num / den), errd = sqrt(numd / den), rel = dev / scale;
  printf("{\"n\": %lld, \"clusters\": %lld, \"batches\": %lld, \"rel_l2_error\": %.3e, "
         "\"fast_vs_parity\": %.3e, \"strict_max_rel\": %.3e, \"ranks2_rel_l2_error\": %.3e}\n",
         (long long)n, (long long)st.n_clusters, (long long)st.n_batches, err, rel, strict, errd);
  return (err < 1e-4 && rel < 1e-13 && strict <= 1e-10 && errd < 1e-4) ? 0 : 2;
}
