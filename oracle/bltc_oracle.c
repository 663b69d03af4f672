/*
 * bltc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-source restatement of the reference BLTC evaluation path
 * (/root/reference/pkg/src/bltc, Python + numba).  It exists to CHECK the CUDA
 * product (paper_2003_01836_b200/csrc) and to time the reference's CPU
 * algorithm on the GPU box's host cores (bench.py cpu_baseline / --impl
 * reference).  Nothing in the product path may link, load or call it.
 *
 * Bit-faithfulness: the reference's numba tiles are compiled without
 * fast-math and without FMA contraction.  This file is built
 * with -O2 -ffp-contract=off -fno-fast-math, uses IEEE sqrt/div and the host
 * libm exp, and follows the reference's operation order exactly, so for
 * Coulomb and the constant kernel it reproduces the reference bit for bit.
 * It is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures, checked in
 * tests/test_oracle_golden.py).
 *
 * Each function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Minimal dynamic-schedule parallel-for over [0, n) on pthreads (the image
 * has no libgomp).  Each worker claims one index at a time, like the
 * reference's ThreadPoolExecutor.map over batches (engine.py:329-334). */
typedef struct {
  int64_t n;
  int64_t next;
  pthread_mutex_t mu;
  void (*body)(void*, int64_t);
  void* arg;
} pfor_t;

static void* pfor_worker(void* p) {
  pfor_t* f = (pfor_t*)p;
  for (;;) {
    pthread_mutex_lock(&f->mu);
    int64_t i = f->next++;
    pthread_mutex_unlock(&f->mu);
    if (i >= f->n) break;
    f->body(f->arg, i);
  }
  return NULL;
}

static void parallel_for(int64_t n, int threads, void (*body)(void*, int64_t), void* arg) {
  if (threads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) body(arg, i);
    return;
  }
  if (threads > 256) threads = 256;
  pfor_t f;
  f.n = n; f.next = 0; f.body = body; f.arg = arg;
  pthread_mutex_init(&f.mu, NULL);
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, pfor_worker, &f);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  pthread_mutex_destroy(&f.mu);
}

#define ORC_SINGULAR_SQ 1e-28                       /* kernels.py:25 */
#define ORC_NODE_TOL 2.2250738585072014e-308         /* interp.py:28 */
#define ORC_DEGENERATE 1e-14                         /* tree.py:30 */

/* ------------------------------------------------------------------------ */
/* Tree / batch partition: tree.py:138-222 (_minimal_bounds, split_dimensions,
 * _split_recursive, _partition, build_source_tree BFS numbering).           */

typedef struct {
  int64_t start, stop;
  double lo[3], hi[3];
  int64_t first_child, next_sibling, n_children; /* temp (recursion) ids */
  int32_t depth;
} tnode;

typedef struct {
  tnode* v;
  int64_t n, cap;
} tnode_vec;

static int64_t tv_push(tnode_vec* tv) {
  if (tv->n == tv->cap) {
    tv->cap = tv->cap ? 2 * tv->cap : 1024;
    tv->v = (tnode*)realloc(tv->v, sizeof(tnode) * tv->cap);
  }
  memset(&tv->v[tv->n], 0, sizeof(tnode));
  tv->v[tv->n].first_child = -1;
  tv->v[tv->n].next_sibling = -1;
  return tv->n++;
}

typedef struct {
  const double *x, *y, *z;
  int64_t* order;
  int64_t* scratch;
  uint8_t* code;
  int64_t max_count;
  tnode_vec tv;
} part_ctx;

/* tree.py:144-177 */
static int64_t split_recursive(part_ctx* c, int64_t start, int64_t stop, int32_t depth) {
  int64_t id = tv_push(&c->tv);
  const double* co[3] = {c->x, c->y, c->z};
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {              /* _minimal_bounds tree.py:138-141 */
    double mn = co[d][c->order[start]], mx = mn;
    for (int64_t i = start + 1; i < stop; ++i) {
      double v = co[d][c->order[i]];
      if (v < mn) mn = v;
      if (v > mx) mx = v;
    }
    lo[d] = mn;
    hi[d] = mx;
  }
  {
    tnode* nd = &c->tv.v[id];
    nd->start = start;
    nd->stop = stop;
    nd->depth = depth;
    memcpy(nd->lo, lo, sizeof lo);
    memcpy(nd->hi, hi, sizeof hi);
  }
  if (stop - start <= c->max_count) return id;
  /* split_dimensions tree.py:56-67 */
  double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  if (ext[0] < ORC_DEGENERATE && ext[1] < ORC_DEGENERATE && ext[2] < ORC_DEGENERATE)
    return id; /* ZeroExtent -> oversized leaf */
  double emax = ext[0];
  if (ext[1] > emax) emax = ext[1];
  if (ext[2] > emax) emax = ext[2];
  double cutoff = emax / sqrt(2.0);
  int dims[3], nd = 0;
  for (int d = 0; d < 3; ++d)
    if (ext[d] > cutoff) dims[nd++] = d;
  double mid[3];
  for (int d = 0; d < 3; ++d) mid[d] = 0.5 * (lo[d] + hi[d]);
  int64_t counts[8] = {0};
  for (int64_t i = start; i < stop; ++i) {
    int64_t p = c->order[i];
    int code = 0;
    for (int k = 0; k < nd; ++k) code = 2 * code + (co[dims[k]][p] >= mid[dims[k]]);
    c->code[i] = (uint8_t)code;
    counts[code]++;
  }
  int nonempty = 0;
  for (int k = 0; k < 8; ++k) nonempty += counts[k] > 0;
  if (nonempty < 2) return id;
  /* stable argsort by code == stable counting sort (tree.py:168) */
  int64_t off[8], acc = 0;
  for (int k = 0; k < 8; ++k) { off[k] = acc; acc += counts[k]; }
  for (int64_t i = start; i < stop; ++i) c->scratch[start + off[c->code[i]]++] = c->order[i];
  memcpy(c->order + start, c->scratch + start, sizeof(int64_t) * (stop - start));
  int64_t offset = start, prev = -1;
  for (int k = 0; k < 8; ++k) {
    if (counts[k] == 0) continue;
    int64_t ch = split_recursive(c, offset, offset + counts[k], depth + 1);
    if (prev < 0) c->tv.v[id].first_child = ch;
    else c->tv.v[prev].next_sibling = ch;
    c->tv.v[id].n_children++;
    prev = ch;
    offset += counts[k];
  }
  return id;
}

typedef struct {
  int64_t n, n_nodes;
  int64_t* order;        /* reordered position -> original index */
  int64_t* start;        /* BFS-numbered nodes (tree.py:198-217) */
  int64_t* stop;
  double* lo;            /* [n_nodes][3] */
  double* hi;
  int64_t* child_start;
  int64_t* child_count;
  int32_t* depth;
  int64_t n_leaves;
  int64_t* leaf_dfs;     /* leaves in DFS order (build_target_batches collect, tree.py:240-250) */
} orc_tree;

static void dfs_leaves(const tnode_vec* tv, const int64_t* bfs_id, int64_t t, int64_t* out, int64_t* k) {
  if (tv->v[t].n_children == 0) { out[(*k)++] = bfs_id[t]; return; }
  for (int64_t ch = tv->v[t].first_child; ch >= 0; ch = tv->v[ch].next_sibling)
    dfs_leaves(tv, bfs_id, ch, out, k);
}

/* _partition (tree.py:180-188) followed by the BFS cluster numbering of
 * build_source_tree (tree.py:198-217). */
orc_tree* orc_partition(int64_t n, const double* x, const double* y, const double* z,
                        int64_t max_count) {
  if (n <= 0 || max_count < 1) return NULL;
  part_ctx c;
  memset(&c, 0, sizeof c);
  c.x = x; c.y = y; c.z = z;
  c.max_count = max_count;
  c.order = (int64_t*)malloc(sizeof(int64_t) * n);
  c.scratch = (int64_t*)malloc(sizeof(int64_t) * n);
  c.code = (uint8_t*)malloc(n);
  for (int64_t i = 0; i < n; ++i) c.order[i] = i;
  split_recursive(&c, 0, n, 0);
  free(c.scratch);
  free(c.code);

  int64_t nn = c.tv.n;
  orc_tree* t = (orc_tree*)calloc(1, sizeof(orc_tree));
  t->n = n;
  t->n_nodes = nn;
  t->order = c.order;
  t->start = (int64_t*)malloc(sizeof(int64_t) * nn);
  t->stop = (int64_t*)malloc(sizeof(int64_t) * nn);
  t->lo = (double*)malloc(sizeof(double) * 3 * nn);
  t->hi = (double*)malloc(sizeof(double) * 3 * nn);
  t->child_start = (int64_t*)calloc(nn, sizeof(int64_t));
  t->child_count = (int64_t*)calloc(nn, sizeof(int64_t));
  t->depth = (int32_t*)malloc(sizeof(int32_t) * nn);
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * nn);   /* temp ids in BFS order */
  int64_t* bfs_id = (int64_t*)malloc(sizeof(int64_t) * nn);  /* temp id -> BFS id */
  int64_t head = 0, tail = 0;
  queue[tail++] = 0;
  while (head < tail) {
    int64_t tmp = queue[head];
    int64_t id = head++;
    bfs_id[tmp] = id;
    const tnode* nd = &c.tv.v[tmp];
    t->start[id] = nd->start;
    t->stop[id] = nd->stop;
    memcpy(t->lo + 3 * id, nd->lo, 3 * sizeof(double));
    memcpy(t->hi + 3 * id, nd->hi, 3 * sizeof(double));
    t->depth[id] = nd->depth;
    if (nd->n_children) {
      t->child_start[id] = tail;
      t->child_count[id] = nd->n_children;
    }
    for (int64_t ch = nd->first_child; ch >= 0; ch = c.tv.v[ch].next_sibling) queue[tail++] = ch;
  }
  int64_t nl = 0;
  for (int64_t i = 0; i < nn; ++i) nl += c.tv.v[i].n_children == 0;
  t->n_leaves = nl;
  t->leaf_dfs = (int64_t*)malloc(sizeof(int64_t) * nl);
  int64_t k = 0;
  dfs_leaves(&c.tv, bfs_id, 0, t->leaf_dfs, &k);
  free(queue);
  free(bfs_id);
  free(c.tv.v);
  return t;
}

int64_t orc_tree_n_nodes(const orc_tree* t) { return t->n_nodes; }
int64_t orc_tree_n_leaves(const orc_tree* t) { return t->n_leaves; }

void orc_tree_export(const orc_tree* t, int64_t* order, int64_t* start, int64_t* stop, double* lo,
                     double* hi, int64_t* child_start, int64_t* child_count, int32_t* depth,
                     int64_t* leaf_dfs) {
  memcpy(order, t->order, sizeof(int64_t) * t->n);
  memcpy(start, t->start, sizeof(int64_t) * t->n_nodes);
  memcpy(stop, t->stop, sizeof(int64_t) * t->n_nodes);
  memcpy(lo, t->lo, sizeof(double) * 3 * t->n_nodes);
  memcpy(hi, t->hi, sizeof(double) * 3 * t->n_nodes);
  memcpy(child_start, t->child_start, sizeof(int64_t) * t->n_nodes);
  memcpy(child_count, t->child_count, sizeof(int64_t) * t->n_nodes);
  memcpy(depth, t->depth, sizeof(int32_t) * t->n_nodes);
  memcpy(leaf_dfs, t->leaf_dfs, sizeof(int64_t) * t->n_leaves);
}

void orc_tree_free(orc_tree* t) {
  if (!t) return;
  free(t->order); free(t->start); free(t->stop); free(t->lo); free(t->hi);
  free(t->child_start); free(t->child_count); free(t->depth); free(t->leaf_dfs);
  free(t);
}

/* BoundingBox.center / .radius (tree.py:46-53): center = 0.5*(lo+hi),
 * radius = 0.5*sqrt(((ex^2 + ey^2) + ez^2)) -- np.sum over 3 elements is
 * sequential left to right. */
void orc_geometry(int64_t n_nodes, const double* lo, const double* hi, double* center,
                  double* radius) {
  for (int64_t i = 0; i < n_nodes; ++i) {
    double e2 = 0.0;
    for (int d = 0; d < 3; ++d) {
      center[3 * i + d] = 0.5 * (lo[3 * i + d] + hi[3 * i + d]);
      double e = hi[3 * i + d] - lo[3 * i + d];
      e2 = d == 0 ? e * e : e2 + e * e;
    }
    radius[i] = 0.5 * sqrt(e2);
  }
}

/* ------------------------------------------------------------------------ */
/* Interaction lists: engine.py:65-130 (mac_accept, _walk, lists_against_root)
 * Output is CSR: per batch, the approx and direct cluster ids in DFS order.  */

typedef struct {
  const double *ccenter, *cradius;
  const int64_t *ccount, *cchild_start, *cchild_count;
  const uint8_t* celig;
  double theta;
  int64_t per_node;
  double bc[3], br;
  int64_t *ap, *dp;         /* output cursors (NULL: count only) */
  int64_t na, nd;
} walk_ctx;

static void walk(walk_ctx* w, int64_t ci) {
  /* mac_accept engine.py:74-85 */
  double dx = w->bc[0] - w->ccenter[3 * ci + 0];
  double dy = w->bc[1] - w->ccenter[3 * ci + 1];
  double dz = w->bc[2] - w->ccenter[3 * ci + 2];
  double dist = sqrt(dx * dx + dy * dy + dz * dz);
  int geom_ok = (w->br + w->cradius[ci] < w->theta * dist);
  if (geom_ok && w->celig[ci]) {
    if (w->per_node < w->ccount[ci]) {     /* accepted */
      if (w->ap) w->ap[w->na] = ci;
      w->na++;
      return;
    }
    if (w->dp) w->dp[w->nd] = ci;          /* SIZE failure -> direct, no recursion */
    w->nd++;
    return;
  }
  if (w->cchild_count[ci] == 0) {           /* geometry failure at a leaf */
    if (w->dp) w->dp[w->nd] = ci;
    w->nd++;
    return;
  }
  for (int64_t k = 0; k < w->cchild_count[ci]; ++k) walk(w, w->cchild_start[ci] + k);
}

/* Two-pass CSR build.  If a_idx/d_idx are NULL only the per-batch counts are
 * written to a_ptr/d_ptr (as exclusive prefix sums, length nb+1). */
void orc_lists(int64_t nb, const double* bcenter, const double* bradius, int64_t nc,
               const double* ccenter, const double* cradius, const int64_t* ccount,
               const uint8_t* celig, const int64_t* cchild_start, const int64_t* cchild_count,
               double theta, int64_t degree, int64_t* a_ptr, int64_t* d_ptr, int64_t* a_idx,
               int64_t* d_idx) {
  (void)nc;
  int64_t per_node = (degree + 1) * (degree + 1) * (degree + 1);
  if (!a_idx) {
    a_ptr[0] = 0;
    d_ptr[0] = 0;
  }
  for (int64_t b = 0; b < nb; ++b) {
    walk_ctx w;
    memset(&w, 0, sizeof w);
    w.ccenter = ccenter; w.cradius = cradius; w.ccount = ccount;
    w.cchild_start = cchild_start; w.cchild_count = cchild_count; w.celig = celig;
    w.theta = theta; w.per_node = per_node;
    w.bc[0] = bcenter[3 * b]; w.bc[1] = bcenter[3 * b + 1]; w.bc[2] = bcenter[3 * b + 2];
    w.br = bradius[b];
    if (a_idx) {
      w.ap = a_idx + a_ptr[b];
      w.dp = d_idx + d_ptr[b];
    }
    walk(&w, 0);
    if (!a_idx) {
      a_ptr[b + 1] = a_ptr[b] + w.na;
      d_ptr[b + 1] = d_ptr[b] + w.nd;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Chebyshev grid of one axis: interp.py:35-56 with the normalised nodes
 * s_k = sin(pi (n-2k) / (2n)) supplied by the caller (numpy on the host). */
static void cheb_points(int degree, double a, double b, const double* s, double* pts) {
  double center = 0.5 * (a + b);
  if (degree == 0) { pts[0] = center; return; }
  double half = 0.5 * (b - a);
  for (int k = 0; k <= degree; ++k) pts[k] = center + half * s[k];
  pts[0] = b;
  pts[degree] = a;
}

void orc_cheb_points(int degree, double a, double b, const double* s, double* pts) {
  cheb_points(degree, a, b, s, pts);
}

/* ------------------------------------------------------------------------ */
/* Upward pass: moments.py:48-115 (_axis_denominator, _intermediate_kernel,
 * _axis_factors, _moments_kernel).  Computes q_hat for the listed clusters. */

static void moments_one(const double* sx, const double* sy, const double* sz, const double* q,
                        int64_t start, int64_t stop, const double* lo, const double* hi,
                        const double* s, const double* w, int degree, double* q_hat) {
  int m = degree + 1;
  double p[3][64];
  for (int d = 0; d < 3; ++d) cheb_points(degree, lo[d], hi[d], s, p[d]);
  int64_t mm = (int64_t)m * m * m;
  for (int64_t k = 0; k < mm; ++k) q_hat[k] = 0.0;
  double t[3][64];
  const double* co[3] = {sx, sy, sz};
  for (int64_t j = start; j < stop; ++j) {
    /* stage 1: _intermediate_kernel moments.py:60-81 */
    double denom = 1.0;
    int hit[3];
    for (int d = 0; d < 3; ++d) {
      double yv = co[d][j], acc = 0.0;
      int h = -1;
      for (int k = 0; k < m; ++k) {               /* _axis_denominator 48-57 */
        double dd = yv - p[d][k];
        if (fabs(dd) < ORC_NODE_TOL) { h = k; acc = 0.0; break; }
        acc += w[k] / dd;
      }
      hit[d] = h;
      if (h < 0) denom *= acc;
    }
    double qt = q[j] / denom;
    /* stage 2: _axis_factors 84-91 and _moments_kernel 94-115 */
    for (int d = 0; d < 3; ++d) {
      double yv = co[d][j];
      if (hit[d] >= 0) {
        for (int k = 0; k < m; ++k) t[d][k] = 0.0;
        t[d][hit[d]] = 1.0;
      } else {
        for (int k = 0; k < m; ++k) t[d][k] = w[k] / (yv - p[d][k]);
      }
    }
    int64_t idx = 0;
    for (int k1 = 0; k1 < m; ++k1) {
      double a = t[0][k1] * qt;
      for (int k2 = 0; k2 < m; ++k2) {
        double b = a * t[1][k2];
        for (int k3 = 0; k3 < m; ++k3) {
          q_hat[idx] += b * t[2][k3];
          idx++;
        }
      }
    }
  }
}

/* Also returns stage-1 values for the reference's compute_intermediate check. */
void orc_intermediate(const double* sx, const double* sy, const double* sz, const double* q,
                      int64_t start, int64_t stop, const double* lo, const double* hi,
                      const double* s, const double* w, int degree, double* qtilde,
                      int64_t* flags) {
  int m = degree + 1;
  double p[3][64];
  for (int d = 0; d < 3; ++d) cheb_points(degree, lo[d], hi[d], s, p[d]);
  const double* co[3] = {sx, sy, sz};
  for (int64_t j = start; j < stop; ++j) {
    double denom = 1.0;
    for (int d = 0; d < 3; ++d) {
      double yv = co[d][j], acc = 0.0;
      int h = -1;
      for (int k = 0; k < m; ++k) {
        double dd = yv - p[d][k];
        if (fabs(dd) < ORC_NODE_TOL) { h = k; break; }
        acc += w[k] / dd;
      }
      flags[3 * (j - start) + d] = h;
      if (h < 0) denom *= acc;
    }
    qtilde[j - start] = q[j] / denom;
  }
}

typedef struct {
  const double *sx, *sy, *sz, *q;
  const int64_t *clusters, *cstart, *cstop;
  const double *lo, *hi, *s, *w;
  int degree;
  double* rows;
} moments_job;

static void moments_body(void* arg, int64_t i) {
  moments_job* J = (moments_job*)arg;
  int64_t mm = (int64_t)(J->degree + 1) * (J->degree + 1) * (J->degree + 1);
  int64_t c = J->clusters[i];
  moments_one(J->sx, J->sy, J->sz, J->q, J->cstart[c], J->cstop[c], J->lo + 3 * c, J->hi + 3 * c,
              J->s, J->w, J->degree, J->rows + i * mm);
}

void orc_moments(const double* sx, const double* sy, const double* sz, const double* q,
                 int64_t n_list, const int64_t* clusters, const int64_t* cstart,
                 const int64_t* cstop, const double* lo, const double* hi, const double* s,
                 const double* w, int degree, double* q_hat_rows, int threads) {
  moments_job J = {sx, sy, sz, q, clusters, cstart, cstop, lo, hi, s, w, degree, q_hat_rows};
  parallel_for(n_list, threads, moments_body, &J);
}

/* ------------------------------------------------------------------------ */
/* Evaluation: engine.py:151-252 (_direct_tile, _approx_tile) driven as in
 * _run_batch / compute_potentials (engine.py:296-335) and, for several source
 * groups, _eval_rank (decomp.py:425-455): per batch, for each group in order:
 * its approx list, then its direct list.                                   */

typedef struct {
  const double *sx, *sy, *sz, *q;   /* that group's reordered sources */
  const int64_t *cstart, *cstop;    /* cluster particle ranges */
  const double *lo, *hi;            /* cluster boxes (for the grids) */
  const int64_t* mrow;              /* cluster -> row in qhat (or -1) */
  const double* qhat;               /* [rows][(n+1)^3] */
  const int64_t *a_ptr, *a_idx, *d_ptr, *d_idx;  /* CSR lists, per target batch */
} orc_group;

static void direct_tile(const double* tx, const double* ty, const double* tz, int64_t i0,
                        int64_t i1, const double* sx, const double* sy, const double* sz,
                        const double* q, int64_t j0, int64_t j1, int kind, double kappa,
                        double* out, double* carry) {
  for (int64_t i = i0; i < i1; ++i) {
    double xi = tx[i], yi = ty[i], zi = tz[i];
    double acc = out[i], comp = carry[i];
    for (int64_t j = j0; j < j1; ++j) {
      double dx = xi - sx[j];
      double dy = yi - sy[j];
      double dz = zi - sz[j];
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 >= ORC_SINGULAR_SQ) {
        double t;
        if (kind == 0) {
          t = q[j] / sqrt(d2);
        } else if (kind == 1) {
          double r = sqrt(d2);
          t = exp(-kappa * r) * q[j] / r;
        } else {
          t = q[j];
        }
        double s = acc + t;
        if (fabs(acc) >= fabs(t)) comp += (acc - s) + t;
        else comp += (t - s) + acc;
        acc = s;
      }
    }
    out[i] = acc;
    carry[i] = comp;
  }
}

static void approx_tile(const double* tx, const double* ty, const double* tz, int64_t i0,
                        int64_t i1, const double* p1, const double* p2, const double* p3, int m,
                        const double* qh, int kind, double kappa, double* out) {
  for (int64_t i = i0; i < i1; ++i) {
    double xi = tx[i], yi = ty[i], zi = tz[i];
    double acc = 0.0;
    int idx = 0;
    for (int k1 = 0; k1 < m; ++k1) {
      double dx = xi - p1[k1];
      for (int k2 = 0; k2 < m; ++k2) {
        double dy = yi - p2[k2];
        for (int k3 = 0; k3 < m; ++k3) {
          if (kind == 2) { acc += qh[idx]; idx++; continue; }
          double dz = zi - p3[k3];
          double d2 = dx * dx + dy * dy + dz * dz;
          if (kind == 0) {
            acc += qh[idx] / sqrt(d2);
          } else {
            double r = sqrt(d2);
            acc += exp(-kappa * r) * qh[idx] / r;
          }
          idx++;
        }
      }
    }
    out[i] += acc;
  }
}

typedef struct {
  const int64_t *sel, *bstart, *bstop;
  const double *tx, *ty, *tz;
  int64_t n_groups;
  const orc_group* groups;
  const double* s;
  int degree, kind;
  double kappa;
  double *out, *carry;
} eval_job;

static void eval_body(void* arg, int64_t ii) {
  eval_job* J = (eval_job*)arg;
  int64_t b = J->sel ? J->sel[ii] : ii;
  int m = J->degree + 1;
  int64_t mm = (int64_t)m * m * m;
  double p[3][64];
  for (int64_t g = 0; g < J->n_groups; ++g) {
    const orc_group* G = &J->groups[g];
    for (int64_t e = G->a_ptr[b]; e < G->a_ptr[b + 1]; ++e) {
      int64_t c = G->a_idx[e];
      for (int d = 0; d < 3; ++d)
        cheb_points(J->degree, G->lo[3 * c + d], G->hi[3 * c + d], J->s, p[d]);
      approx_tile(J->tx, J->ty, J->tz, J->bstart[b], J->bstop[b], p[0], p[1], p[2], m,
                  G->qhat + G->mrow[c] * mm, J->kind, J->kappa, J->out);
    }
    for (int64_t e = G->d_ptr[b]; e < G->d_ptr[b + 1]; ++e) {
      int64_t c = G->d_idx[e];
      direct_tile(J->tx, J->ty, J->tz, J->bstart[b], J->bstop[b], G->sx, G->sy, G->sz, G->q,
                  G->cstart[c], G->cstop[c], J->kind, J->kappa, J->out, J->carry);
    }
  }
}

/* out/carry: zero-initialised by the caller (length = number of targets in the
 * reordered target array).  Batches run in parallel on disjoint output
 * slices, exactly as compute_potentials' thread pool (engine.py:324-334);
 * sel != NULL restricts the run to the listed batches (bounded CPU samples). */
void orc_evaluate(int64_t nb, const int64_t* sel, const int64_t* bstart, const int64_t* bstop,
                  const double* tx, const double* ty, const double* tz, int64_t n_groups,
                  const orc_group* groups, const double* s, int degree, int kind, double kappa,
                  double* out, double* carry, int threads) {
  eval_job J = {sel, bstart, bstop, tx, ty, tz, n_groups, groups, s, degree, kind, kappa, out,
                carry};
  parallel_for(nb, threads, eval_body, &J);
}

/* ------------------------------------------------------------------------ */
/* Brute-force sampled oracle: cli.py:73-127 (_oracle_kernel), Neumaier. */
typedef struct {
  const int64_t* idx;
  const double *tx, *ty, *tz;
  int64_t ns;
  const double *sx, *sy, *sz, *q;
  int kind;
  double kappa;
  double* out;
} dsum_job;

static void dsum_body(void* arg, int64_t a) {
  dsum_job* J = (dsum_job*)arg;
  int64_t i = J->idx[a];
  double acc = 0.0, comp = 0.0;
  double xi = J->tx[i], yi = J->ty[i], zi = J->tz[i];
  for (int64_t j = 0; j < J->ns; ++j) {
    double dx = xi - J->sx[j];
    double dy = yi - J->sy[j];
    double dz = zi - J->sz[j];
    double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 >= ORC_SINGULAR_SQ) {
      double t;
      if (J->kind == 0) t = J->q[j] / sqrt(d2);
      else if (J->kind == 1) { double r = sqrt(d2); t = exp(-J->kappa * r) * J->q[j] / r; }
      else t = J->q[j];
      double s = acc + t;
      if (fabs(acc) >= fabs(t)) comp += (acc - s) + t;
      else comp += (t - s) + acc;
      acc = s;
    }
  }
  J->out[a] = acc + comp;
}

void orc_direct_sum(int64_t n_idx, const int64_t* idx, const double* tx, const double* ty,
                    const double* tz, int64_t ns, const double* sx, const double* sy,
                    const double* sz, const double* q, int kind, double kappa, double* out,
                    int threads) {
  dsum_job J = {idx, tx, ty, tz, ns, sx, sy, sz, q, kind, kappa, out};
  parallel_for(n_idx, threads, dsum_body, &J);
}
