/* dipole_oracle.c — CPU restatement of the reference's Barnes-Hut dipole-sum
 * hot path. TEST INFRASTRUCTURE ONLY (see dipole_oracle.h): the checker for
 * the CUDA path, never part of it.
 *
 * Paths cited are relative to /root/reference/proj. Compile with
 * -ffp-contract=off (oracle/Makefile) so no FMA contraction changes rounding.
 */
#include "dipole_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

static const double kInvFourPi = 0.07957747154594766788444188168625718101; /* util.hpp:17-19 */
static const double kSqrtPi = 1.77245385090551602729816748334114518;
enum { STACK_CAP = 2048 }; /* bhtree.cpp:185 */

/* ---------------------------------------------------------------- vectors */
/* Eigen squaredNorm / dot association for 3-vectors: (x*x + y*y) + z*z. */
static inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

/* ---------------------------------------------------------- kernel math */
/* erf_series: kernels.cpp:12-24 */
static double erf_series(double x, double expmx2) {
  double x2 = x * x, term = x, sum = x, denom = 1.0;
  for (int n = 1; n < 80; ++n) {
    denom += 2.0;
    term *= 2.0 * x2 / denom;
    sum += term;
    if (term < 1e-18 * sum) break;
  }
  return 2.0 / kSqrtPi * expmx2 * sum;
}

/* erfc_cf (modified Lentz): kernels.cpp:28-45 */
static double erfc_cf(double x, double expmx2) {
  const double tiny = 1e-300;
  double c = 1.0 / tiny, d = 1.0 / x, h = d;
  for (int i = 1; i < 300; ++i) {
    double a = i / 2.0;
    d = x + a * d;
    if (fabs(d) < tiny) d = tiny;
    c = x + a / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    double delta = d * c;
    h *= delta;
    if (fabs(delta - 1.0) < 1e-17) break;
  }
  return expmx2 / kSqrtPi * h;
}

/* tau_derivs: kernels.cpp:49-61 */
static void tau_derivs(double t, int order, double* tv, double* tp, double* ts) {
  if (t >= 6.5) {
    *tv = 1.0;
    if (order >= 1) *tp = 0.0;
    if (order >= 2) *ts = 0.0;
    return;
  }
  double u = exp(-t * t);
  double e = t <= 2.0 ? erf_series(t, u) : 1.0 - erfc_cf(t, u);
  *tv = e - 2.0 * t / kSqrtPi * u;
  if (order >= 1) *tp = 4.0 * t * t / kSqrtPi * u;
  if (order >= 2) *ts = 8.0 / kSqrtPi * (t - t * t * t) * u;
}

/* erf_approx: kernels.cpp:65-75 */
double ora_erf(double x) {
  double ax = fabs(x), v;
  if (ax <= 2.0)
    v = erf_series(ax, exp(-ax * ax));
  else if (ax < 6.5)
    v = 1.0 - erfc_cf(ax, exp(-ax * ax));
  else
    v = 1.0;
  return x < 0 ? -v : v;
}

/* tau: kernels.cpp:77-79 */
double ora_tau(double t) { return ora_erf(t) - 2.0 * t / kSqrtPi * exp(-t * t); }

/* normal_cdf / normal_pdf / normal_hazard: kernels.cpp:89-98 */
static double normal_cdf(double z) { return 0.5 * (1.0 + ora_erf(z * 0.7071067811865475244)); }
static double normal_pdf(double z) { return exp(-0.5 * z * z) * 0.3989422804014326779; }
double ora_normal_hazard(double z) {
  if (z > -6.0) return normal_pdf(z) / normal_cdf(z);
  double z2 = z * z;
  return -z / (1.0 - 1.0 / z2 + 3.0 / (z2 * z2) - 15.0 / (z2 * z2 * z2));
}

typedef struct {
  double W, Wp_r, dW_de, dWp_r_de, R, Rp_r, dR_de;
} coeffs;

/* kernel_coeffs: kernels.cpp:100-153 */
static coeffs kernel_coeffs(double r, const ora_params* p, int order) {
  coeffs k = {0, 0, 0, 0, 0, 0, 0};
  if (p->desingularized) { /* :102-111 */
    double d2 = p->desing_delta * p->desing_delta;
    double s = r * r + d2;
    double s32 = pow(s, 1.5);
    k.W = 1.0 / s32;
    k.Wp_r = -3.0 / (s32 * s);
    k.R = r / s32;
    k.Rp_r = (r > 0) ? (1.0 / s32 - 3.0 * r * r / (s32 * s)) / r : 0.0;
    return k;
  }
  double eps = p->epsilon;
  if (eps <= 0.0) { /* singular, :112-121 */
    double r2 = r * r, r3 = r2 * r;
    k.W = 1.0 / r3;
    k.Wp_r = -3.0 / (r3 * r2);
    k.R = 1.0 / r2;
    k.Rp_r = -2.0 / (r2 * r2);
    return k;
  }
  double t = r / eps;
  double e3 = eps * eps * eps;
  double c = 2.0 / (kSqrtPi * e3);
  if (t < 0.05) { /* series, :125-136 */
    double t2 = t * t, t4 = t2 * t2;
    k.W = c * (2.0 / 3.0 - 0.4 * t2 + t4 / 7.0);
    k.Wp_r = c / (eps * eps) * (-0.8 + (4.0 / 7.0) * t2 - (2.0 / 9.0) * t4);
    k.dWp_r_de = c / e3 * (4.0 - 4.0 * t2 + 2.0 * t4);
    k.dW_de = -2.0 * c / eps * (1.0 - t2 + 0.5 * t4);
    k.R = k.W * r;
    k.dR_de = k.dW_de * r;
    if (r > 0) k.Rp_r = 2.0 * c / r * (1.0 / 3.0 - 0.6 * t2 + (5.0 / 14.0) * t4);
    return k;
  }
  double r2 = r * r, r3 = r2 * r, r4 = r2 * r2; /* closed form, :137-151 */
  double tv = 0, tp = 0, ts = 0;
  tau_derivs(t, order, &tv, &tp, &ts);
  double e2 = eps * eps;
  k.W = tv / r3;
  k.R = tv / r2;
  if (order >= 1) {
    k.Wp_r = tp / (eps * r4) - 3.0 * tv / (r4 * r);
    k.Rp_r = tp / (eps * r3) - 2.0 * tv / r4;
  }
  if (order >= 2) {
    k.dW_de = -tp / (e2 * r2);
    k.dWp_r_de = -ts / (e2 * eps * r3) + 2.0 * tp / (e2 * r4);
    k.dR_de = -tp / (e2 * r);
  }
  return k;
}

void ora_kernel_coeffs(double r, const ora_params* p, int order, double* o) {
  coeffs k = kernel_coeffs(r, p, order);
  o[0] = k.W, o[1] = k.Wp_r, o[2] = k.dW_de, o[3] = k.dWp_r_de;
  o[4] = k.R, o[5] = k.Rp_r, o[6] = k.dR_de;
}

/* ------------------------------------------------------------------ tree */
struct ora_tree {
  int64_t n, nodes, cap;
  int C, max_leaf, max_depth;
  double *ctr, *area, *radius;        /* nodes x 3, nodes, nodes */
  int32_t *begin, *end, *cbeg, *ccnt, *parent;
  uint8_t* leaf;
  double *tcenter, *thalf;            /* BFS task data (bhtree.cpp:52-57) */
  int32_t* tdepth;
  int32_t *order, *leaf_of;
  double *pos, *nrm, *ar, *mu;        /* SoA mirrors, refresh_point_data :20-34 */
  uint8_t* kinds;                      /* 0 Dipole, 1 Radial */
  double *mv, *ms;                     /* moments_v_ nodes x C x 3, moments_s_ nodes x C */
};

static void* xrealloc(void* p, size_t n) {
  void* q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}

static int32_t push_node(ora_tree* t) {
  if (t->nodes == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 1024;
    size_t c = (size_t)t->cap;
    t->ctr = xrealloc(t->ctr, c * 3 * sizeof(double));
    t->area = xrealloc(t->area, c * sizeof(double));
    t->radius = xrealloc(t->radius, c * sizeof(double));
    t->begin = xrealloc(t->begin, c * sizeof(int32_t));
    t->end = xrealloc(t->end, c * sizeof(int32_t));
    t->cbeg = xrealloc(t->cbeg, c * sizeof(int32_t));
    t->ccnt = xrealloc(t->ccnt, c * sizeof(int32_t));
    t->parent = xrealloc(t->parent, c * sizeof(int32_t));
    t->leaf = xrealloc(t->leaf, c);
    t->tcenter = xrealloc(t->tcenter, c * 3 * sizeof(double));
    t->thalf = xrealloc(t->thalf, c * sizeof(double));
    t->tdepth = xrealloc(t->tdepth, c * sizeof(int32_t));
  }
  int32_t i = (int32_t)t->nodes++;
  t->ctr[3 * i] = t->ctr[3 * i + 1] = t->ctr[3 * i + 2] = 0;
  t->area[i] = t->radius[i] = 0;
  t->begin[i] = t->end[i] = t->cbeg[i] = t->ccnt[i] = 0;
  t->parent[i] = -1;
  t->leaf[i] = 0;
  return i;
}

/* refresh_point_data: bhtree.cpp:20-34 */
static void refresh_point_data(ora_tree* t, const double* pos, const double* nrm,
                               const double* area, const double* mu) {
  size_t n = (size_t)t->n;
  memcpy(t->pos, pos, n * 3 * sizeof(double));
  memcpy(t->nrm, nrm, n * 3 * sizeof(double));
  memcpy(t->ar, area, n * sizeof(double));
  memcpy(t->mu, mu, n * (size_t)t->C * sizeof(double));
}

/* build_structure: bhtree.cpp:36-105. The FIFO queue visits nodes in creation
 * order, so node index doubles as the queue cursor. */
static void build_structure(ora_tree* t) {
  int64_t m = t->n;
  t->nodes = 0;
  for (int64_t i = 0; i < m; ++i) t->order[i] = (int32_t)i, t->leaf_of[i] = -1;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = t->pos[a];
  for (int64_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) { /* cwiseMin / cwiseMax (:44-47) */
      double v = t->pos[3 * i + a];
      if (v < lo[a]) lo[a] = v;
      if (hi[a] < v) hi[a] = v;
    }
  double rc[3], ext[3];
  for (int a = 0; a < 3; ++a) rc[a] = 0.5 * (lo[a] + hi[a]), ext[a] = hi[a] - lo[a];
  double mx = ext[0]; /* maxCoeff */
  if (mx < ext[1]) mx = ext[1];
  if (mx < ext[2]) mx = ext[2];
  double root_half = 0.5 * mx;
  root_half = root_half > 0 ? root_half * (1.0 + 1e-7) : 1.0; /* :50 */
  int32_t r = push_node(t);
  t->begin[r] = 0, t->end[r] = (int32_t)m;
  memcpy(t->tcenter, rc, sizeof rc);
  t->thalf[0] = root_half, t->tdepth[0] = 0;
  int32_t* bucket = xrealloc(NULL, (size_t)m * sizeof(int32_t));
  int32_t* oct = xrealloc(NULL, (size_t)m * sizeof(int32_t));
  for (int64_t ni = 0; ni < t->nodes; ++ni) {
    int32_t b = t->begin[ni], e = t->end[ni];
    if (e - b <= t->max_leaf || t->tdepth[ni] >= t->max_depth) { /* :69-72 */
      t->leaf[ni] = 1;
      continue;
    }
    const double* c = t->tcenter + 3 * ni;
    int32_t counts[8] = {0};
    for (int32_t j = b; j < e; ++j) { /* octant, :77-78 */
      const double* q = t->pos + 3 * (int64_t)t->order[j];
      int o = (q[0] >= c[0] ? 1 : 0) | (q[1] >= c[1] ? 2 : 0) | (q[2] >= c[2] ? 4 : 0);
      oct[j] = o;
      counts[o]++;
    }
    int32_t off[8], w = 0;
    for (int o = 0; o < 8; ++o) off[o] = w, w += counts[o];
    for (int32_t j = b; j < e; ++j) bucket[off[oct[j]]++] = t->order[j]; /* stable partition */
    memcpy(t->order + b, bucket, (size_t)(e - b) * sizeof(int32_t));
    int32_t child_begin = (int32_t)t->nodes, child_count = 0, write = b;
    double half = t->thalf[ni];
    int32_t depth = t->tdepth[ni];
    for (int o = 0; o < 8; ++o) { /* children in octant order, empty skipped (:84-97) */
      if (!counts[o]) continue;
      int32_t ci = push_node(t);
      c = t->tcenter + 3 * ni; /* push_node may have moved the arrays */
      t->begin[ci] = write;
      write += counts[o];
      t->end[ci] = write;
      t->parent[ci] = (int32_t)ni;
      double hh = 0.5 * half; /* 0.5 * t.half * (+-1) is exact (:93-94) */
      t->tcenter[3 * ci + 0] = c[0] + hh * ((o & 1) ? 1.0 : -1.0);
      t->tcenter[3 * ci + 1] = c[1] + hh * ((o & 2) ? 1.0 : -1.0);
      t->tcenter[3 * ci + 2] = c[2] + hh * ((o & 4) ? 1.0 : -1.0);
      t->thalf[ci] = 0.5 * half;
      t->tdepth[ci] = depth + 1;
      ++child_count;
    }
    t->cbeg[ni] = child_begin;
    t->ccnt[ni] = child_count;
  }
  free(bucket);
  free(oct);
  for (int64_t ni = 0; ni < t->nodes; ++ni) /* point_leaf, :101-104 */
    if (t->leaf[ni])
      for (int32_t j = t->begin[ni]; j < t->end[ni]; ++j) t->leaf_of[t->order[j]] = (int32_t)ni;
}

/* compute_node_geometry: bhtree.cpp:107-134 */
static void compute_node_geometry(ora_tree* t) {
  for (int64_t ni = 0; ni < t->nodes; ++ni) {
    int32_t b = t->begin[ni], e = t->end[ni];
    double* ctr = t->ctr + 3 * ni;
    if (e - b == 1) {
      int64_t p = t->order[b];
      t->area[ni] = t->ar[p];
      memcpy(ctr, t->pos + 3 * p, 3 * sizeof(double));
      t->radius[ni] = 0.0;
      continue;
    }
    double asum = 0, psum[3] = {0, 0, 0}, mean[3] = {0, 0, 0};
    for (int32_t j = b; j < e; ++j) {
      int64_t p = t->order[j];
      asum += t->ar[p];
      for (int a = 0; a < 3; ++a) psum[a] += t->ar[p] * t->pos[3 * p + a];
      for (int a = 0; a < 3; ++a) mean[a] += t->pos[3 * p + a];
    }
    t->area[ni] = asum;
    for (int a = 0; a < 3; ++a)
      ctr[a] = asum > 0 ? psum[a] / asum : mean[a] / (double)(e - b);
    double r2max = 0;
    for (int32_t j = b; j < e; ++j) {
      const double* q = t->pos + 3 * (int64_t)t->order[j];
      double d[3] = {q[0] - ctr[0], q[1] - ctr[1], q[2] - ctr[2]};
      double s = dot3(d, d);
      r2max = r2max < s ? s : r2max; /* std::max(r2max, s) */
    }
    t->radius[ni] = sqrt(r2max);
  }
}

/* compute_node_moments: bhtree.cpp:136-156 */
static void compute_node_moments(ora_tree* t) {
  const int C = t->C;
  size_t nn = (size_t)t->nodes * C;
  t->mv = xrealloc(t->mv, nn * 3 * sizeof(double));
  t->ms = xrealloc(t->ms, nn * sizeof(double));
  memset(t->mv, 0, nn * 3 * sizeof(double));
  memset(t->ms, 0, nn * sizeof(double));
  for (int64_t ni = 0; ni < t->nodes; ++ni) {
    if (!(t->area[ni] > 0)) continue;
    double* mv = t->mv + (size_t)ni * C * 3;
    double* ms = t->ms + (size_t)ni * C;
    for (int32_t j = t->begin[ni]; j < t->end[ni]; ++j) {
      int64_t p = t->order[j];
      for (int c = 0; c < C; ++c) {
        double am = t->ar[p] * t->mu[p * C + c];
        for (int a = 0; a < 3; ++a) mv[3 * c + a] += am * t->nrm[3 * p + a];
        ms[c] += am;
      }
    }
    for (int c = 0; c < C; ++c) {
      for (int a = 0; a < 3; ++a) mv[3 * c + a] /= t->area[ni];
      ms[c] /= t->area[ni];
    }
  }
}

/* DipoleTree::build: bhtree.cpp:158-169 */
ora_tree* ora_tree_build(const double* pos, const double* nrm, const double* area,
                         const double* mu, int64_t n, int32_t C, int32_t max_leaf,
                         int32_t max_depth) {
  if (n <= 0 || C <= 0) return NULL; /* DataError: empty cloud */
  ora_tree* t = calloc(1, sizeof(ora_tree));
  t->n = n;
  t->C = C;
  t->max_leaf = max_leaf < 1 ? 1 : max_leaf;
  t->max_depth = max_depth < 0 ? 0 : max_depth;
  t->pos = xrealloc(NULL, (size_t)n * 3 * sizeof(double));
  t->nrm = xrealloc(NULL, (size_t)n * 3 * sizeof(double));
  t->ar = xrealloc(NULL, (size_t)n * sizeof(double));
  t->mu = xrealloc(NULL, (size_t)n * C * sizeof(double));
  t->order = xrealloc(NULL, (size_t)n * sizeof(int32_t));
  t->leaf_of = xrealloc(NULL, (size_t)n * sizeof(int32_t));
  t->kinds = calloc((size_t)C, 1); /* channel_kernels_ all Dipole (:164) */
  refresh_point_data(t, pos, nrm, area, mu);
  build_structure(t);
  compute_node_geometry(t);
  compute_node_moments(t);
  return t;
}

void ora_tree_free(ora_tree* t) {
  if (!t) return;
  void* ps[] = {t->ctr, t->area, t->radius, t->begin, t->end, t->cbeg, t->ccnt, t->parent,
                t->leaf, t->tcenter, t->thalf, t->tdepth, t->order, t->leaf_of, t->pos, t->nrm,
                t->ar, t->mu, t->kinds, t->mv, t->ms};
  for (size_t i = 0; i < sizeof ps / sizeof ps[0]; ++i) free(ps[i]);
  free(t);
}

/* update_moments: bhtree.cpp:171-176 */
int ora_tree_update_moments(ora_tree* t, const double* pos, const double* nrm, const double* area,
                            const double* mu, int64_t n, int32_t C) {
  if (n != t->n || C != t->C) return 2; /* DataError */
  refresh_point_data(t, pos, nrm, area, mu);
  compute_node_moments(t);
  return 0;
}

/* set_channel_kernels: bhtree.cpp:178-182 */
int ora_tree_set_kinds(ora_tree* t, const uint8_t* kinds, int32_t C) {
  if (C != t->C) return 2;
  memcpy(t->kinds, kinds, (size_t)C);
  return 0;
}

int64_t ora_tree_node_count(const ora_tree* t) { return t->nodes; }

void ora_tree_export(const ora_tree* t, double* geo, int32_t* topo, int32_t* order,
                     int32_t* leaf_of) {
  for (int64_t i = 0; i < t->nodes; ++i) {
    if (geo) {
      geo[5 * i] = t->ctr[3 * i], geo[5 * i + 1] = t->ctr[3 * i + 1];
      geo[5 * i + 2] = t->ctr[3 * i + 2], geo[5 * i + 3] = t->area[i];
      geo[5 * i + 4] = t->radius[i];
    }
    if (topo) {
      int32_t* s = topo + 6 * i;
      s[0] = t->begin[i], s[1] = t->end[i], s[2] = t->cbeg[i], s[3] = t->ccnt[i];
      s[4] = t->parent[i], s[5] = t->leaf[i];
    }
  }
  if (order) memcpy(order, t->order, (size_t)t->n * sizeof(int32_t));
  if (leaf_of) memcpy(leaf_of, t->leaf_of, (size_t)t->n * sizeof(int32_t));
}

void ora_tree_export_moments(const ora_tree* t, double* mv, double* ms) {
  size_t nn = (size_t)t->nodes * t->C;
  if (mv) memcpy(mv, t->mv, nn * 3 * sizeof(double));
  if (ms) memcpy(ms, t->ms, nn * sizeof(double));
}

/* ------------------------------------------------------------ parallel_for */
typedef struct {
  void (*body)(void* ctx, int64_t lo, int64_t hi, int w);
  void* ctx;
  int64_t lo, hi;
  int w;
} pf_task;

static void* pf_run(void* a) {
  pf_task* t = a;
  t->body(t->ctx, t->lo, t->hi, t->w);
  return NULL;
}

/* Deterministic chunking as util.cpp:7-26: chunk w goes to worker w. */
static int parallel_for(int64_t n, int workers, void (*body)(void*, int64_t, int64_t, int),
                        void* ctx) {
  if (n <= 0) return 0;
  if (workers < 1) workers = 1;
  if (workers > n) workers = (int)n;
  if (workers == 1) {
    body(ctx, 0, n, 0);
    return 1;
  }
  int64_t chunk = (n + workers - 1) / workers;
  pthread_t* th = xrealloc(NULL, sizeof(pthread_t) * (size_t)workers);
  pf_task* tk = xrealloc(NULL, sizeof(pf_task) * (size_t)workers);
  int used = 0;
  for (int w = 0; w < workers; ++w) {
    int64_t lo = w * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo >= hi) break;
    tk[w] = (pf_task){body, ctx, lo, hi, w};
    pthread_create(&th[w], NULL, pf_run, &tk[w]);
    ++used;
  }
  for (int w = 0; w < used; ++w) pthread_join(th[w], NULL);
  free(th);
  free(tk);
  return used;
}

/* ------------------------------------------------------------ traversals */
static inline int is_near(double r, const ora_params* p) {
  return !p->desingularized && p->epsilon > 0 && r / p->epsilon < 6.5;
}

/* primal (bhtree.cpp:188-234), primal_channel (:236-274) and
 * primal_with_gradient (:276-334) for one query. */
/* out_abs (nc) / grad_abs (3C), test-only and NULL normally: the sum of |terms|
 * each output accumulated (the tolerance scale of a parity test where the
 * sum cancels); the outputs are unaffected. */
static void primal_one_mag(const ora_tree* t, const ora_params* p, double beta, const double* x,
                           int mode, int channel, double* out, double* grad, ora_counters* cnt,
                           double* out_abs, double* grad_abs) {
  const int C = t->C;
  int nc = mode == 2 ? 1 : C;
  for (int c = 0; c < nc; ++c) out[c] = 0.0;
  if (grad)
    for (int c = 0; c < 3 * C; ++c) grad[c] = 0.0;
  if (out_abs)
    for (int c = 0; c < nc; ++c) out_abs[c] = 0.0;
  if (grad_abs)
    for (int c = 0; c < 3 * C; ++c) grad_abs[c] = 0.0;
  double beta2 = beta * beta;
  int singular = p->epsilon <= 0.0 && !p->desingularized;
  int order = mode == 1 ? 1 : 0;
  int32_t stack[STACK_CAP];
  int sp = 0;
  stack[sp++] = 0;
  while (sp) {
    int32_t ni = stack[--sp];
    if (cnt) cnt->visited++;
    const double* ctr = t->ctr + 3 * ni;
    double d[3] = {ctr[0] - x[0], ctr[1] - x[1], ctr[2] - x[2]};
    double dist2 = dot3(d, d);
    if (dist2 > beta2 * t->radius[ni] * t->radius[ni]) { /* strict test, :204 */
      if (!(t->area[ni] > 0)) continue;
      double rr = sqrt(dist2);
      coeffs k = kernel_coeffs(rr, p, order);
      if (cnt) { if (is_near(rr, p)) cnt->far_near++; else cnt->far_far++; }
      double A = t->area[ni] * kInvFourPi;
      for (int c = 0; c < C; ++c) {
        if (mode == 2 && c != channel) continue;
        double* o = mode == 2 ? out : out + c;
        const double* v = t->mv + ((size_t)ni * C + c) * 3;
        double s = t->ms[(size_t)ni * C + c];
        double* oa = out_abs ? (mode == 2 ? out_abs : out_abs + c) : NULL;
        if (t->kinds[c] == 0) {
          double vd = dot3(v, d);
          *o += A * k.W * vd;
          if (oa) *oa += fabs(A * k.W * vd);
          if (mode == 1)
            for (int a = 0; a < 3; ++a) grad[3 * c + a] -= A * (k.W * v[a] + k.Wp_r * vd * d[a]);
          if (mode == 1 && grad_abs)
            for (int a = 0; a < 3; ++a)
              grad_abs[3 * c + a] += fabs(A) * (fabs(k.W * v[a]) + fabs(k.Wp_r * vd * d[a]));
        } else {
          *o += A * k.R * s;
          if (oa) *oa += fabs(A * k.R * s);
          if (mode == 1)
            for (int a = 0; a < 3; ++a) grad[3 * c + a] -= A * k.Rp_r * s * d[a];
          if (mode == 1 && grad_abs)
            for (int a = 0; a < 3; ++a) grad_abs[3 * c + a] += fabs(A * k.Rp_r * s * d[a]);
        }
      }
    } else if (t->leaf[ni]) {
      for (int32_t j = t->begin[ni]; j < t->end[ni]; ++j) {
        int64_t pi = t->order[j];
        const double* pp = t->pos + 3 * pi;
        const double* nn = t->nrm + 3 * pi;
        double dm[3] = {pp[0] - x[0], pp[1] - x[1], pp[2] - x[2]};
        double r2 = dot3(dm, dm);
        if (r2 == 0.0 && (singular || mode == 1)) continue; /* :219, :316 */
        double rr = sqrt(r2);
        coeffs k = kernel_coeffs(rr, p, order);
        if (cnt) { if (is_near(rr, p)) cnt->pt_near++; else cnt->pt_far++; }
        double ndot = dot3(nn, dm);
        for (int c = 0; c < C; ++c) {
          if (mode == 2 && c != channel) continue;
          double* o = mode == 2 ? out : out + c;
          double A = t->ar[pi] * kInvFourPi * t->mu[pi * C + c];
          double* oa = out_abs ? (mode == 2 ? out_abs : out_abs + c) : NULL;
          if (t->kinds[c] == 0) {
            *o += A * k.W * ndot;
            if (oa) *oa += fabs(A * k.W * ndot);
            if (mode == 1)
              for (int a = 0; a < 3; ++a) grad[3 * c + a] -= A * (k.W * nn[a] + k.Wp_r * ndot * dm[a]);
            if (mode == 1 && grad_abs)
              for (int a = 0; a < 3; ++a)
                grad_abs[3 * c + a] += fabs(A) * (fabs(k.W * nn[a]) + fabs(k.Wp_r * ndot * dm[a]));
          } else {
            *o += A * k.R;
            if (oa) *oa += fabs(A * k.R);
            if (mode == 1)
              for (int a = 0; a < 3; ++a) grad[3 * c + a] -= A * k.Rp_r * dm[a];
            if (mode == 1 && grad_abs)
              for (int a = 0; a < 3; ++a) grad_abs[3 * c + a] += fabs(A * k.Rp_r * dm[a]);
          }
        }
      }
    } else {
      for (int32_t c = 0; c < t->ccnt[ni]; ++c) stack[sp++] = t->cbeg[ni] + c;
    }
  }
}

static void primal_one(const ora_tree* t, const ora_params* p, double beta, const double* x,
                       int mode, int channel, double* out, double* grad, ora_counters* cnt) {
  primal_one_mag(t, p, beta, x, mode, channel, out, grad, cnt, NULL, NULL);
}

typedef struct {
  const ora_tree* t;
  const ora_params* p;
  double beta;
  const double* xs;
  int mode, channel;
  double *out, *grad;
  ora_counters* cnt;
  double *out_abs, *grad_abs;
} primal_ctx;

static void primal_body(void* v, int64_t lo, int64_t hi, int w) {
  (void)w;
  primal_ctx* c = v;
  const int C = c->t->C;
  int nc = c->mode == 2 ? 1 : C;
  for (int64_t i = lo; i < hi; ++i) {
    ora_counters k = {0, 0, 0, 0, 0};
    primal_one_mag(c->t, c->p, c->beta, c->xs + 3 * i, c->mode, c->channel, c->out + i * nc,
                   c->grad ? c->grad + i * C * 3 : NULL, c->cnt ? &k : NULL,
                   c->out_abs ? c->out_abs + i * nc : NULL,
                   c->grad_abs ? c->grad_abs + i * C * 3 : NULL);
    if (c->cnt) c->cnt[i] = k;
  }
}

void ora_primal_ex(const ora_tree* t, const ora_params* p, double beta, const double* xs,
                   int64_t q, int mode, int channel, double* out, double* grad,
                   ora_counters* counters, int threads, double* out_abs, double* grad_abs) {
  primal_ctx c = {t, p, beta, xs, mode, channel, out, mode == 1 ? grad : NULL, counters,
                  out_abs, mode == 1 ? grad_abs : NULL};
  parallel_for(q, threads, primal_body, &c);
}

void ora_primal(const ora_tree* t, const ora_params* p, double beta, const double* xs, int64_t q,
                int mode, int channel, double* out, double* grad, ora_counters* counters,
                int threads) {
  ora_primal_ex(t, p, beta, xs, q, mode, channel, out, grad, counters, threads, NULL, NULL);
}

/* GradientBuffer (bhtree.hpp:40-49). Test-only extension (mag != 0): beside
 * every accumulator, a bound on the SUM OF ABSOLUTE VALUES of the terms that
 * reach it (vector terms by their Euclidean norm), so a parity test can scale
 * its tolerance to the cancellation the reference's own sum went through.
 * The accumulators themselves are untouched by it. */
typedef struct {
  double *node_v, *node_s, *point_mu, *point_n, d_eps;
  int mag;
  double *node_va, *node_sa, *point_mua, *point_na, d_epsa;
} gradbuf;

static void gradbuf_init(gradbuf* b, const ora_tree* t) {
  size_t nn = (size_t)t->nodes * t->C, np = (size_t)t->n * t->C;
  b->node_v = calloc(nn * 3, sizeof(double));
  b->node_s = calloc(nn, sizeof(double));
  b->point_mu = calloc(np, sizeof(double));
  b->point_n = calloc((size_t)t->n * 3, sizeof(double));
  b->d_eps = 0;
  b->mag = 0;
  b->node_va = b->node_sa = b->point_mua = b->point_na = NULL;
  b->d_epsa = 0;
}

static void gradbuf_init_mag(gradbuf* b, const ora_tree* t) {
  size_t nn = (size_t)t->nodes * t->C, np = (size_t)t->n * t->C;
  gradbuf_init(b, t);
  b->mag = 1;
  b->node_va = calloc(nn, sizeof(double));
  b->node_sa = calloc(nn, sizeof(double));
  b->point_mua = calloc(np, sizeof(double));
  b->point_na = calloc((size_t)t->n * 3, sizeof(double));
}

static void gradbuf_free(gradbuf* b) {
  free(b->node_v), free(b->node_s), free(b->point_mu), free(b->point_n);
  free(b->node_va), free(b->node_sa), free(b->point_mua), free(b->point_na);
}

static inline double norm3(const double* a) { return sqrt(dot3(a, a)); }

/* adjoint: bhtree.cpp:345-417 */
static void adjoint_one(const ora_tree* t, const ora_params* p, double beta, const double* x,
                        const double* d_out, const double* d_grad, gradbuf* buf) {
  const int C = t->C;
  double beta2 = beta * beta;
  int with_grad = d_grad != NULL;
  int32_t stack[STACK_CAP];
  int sp = 0;
  stack[sp++] = 0;
  while (sp) {
    int32_t ni = stack[--sp];
    const double* ctr = t->ctr + 3 * ni;
    double d[3] = {ctr[0] - x[0], ctr[1] - x[1], ctr[2] - x[2]};
    double dist2 = dot3(d, d);
    if (dist2 > beta2 * t->radius[ni] * t->radius[ni]) {
      if (!(t->area[ni] > 0)) continue;
      coeffs k = kernel_coeffs(sqrt(dist2), p, 2);
      double A = t->area[ni] * kInvFourPi;
      for (int c = 0; c < C; ++c) {
        double ds = d_out[c];
        if (t->kinds[c] == 0) {
          double dv[3];
          for (int a = 0; a < 3; ++a) dv[a] = A * k.W * ds * d[a];
          const double* v = t->mv + ((size_t)ni * C + c) * 3;
          double vd = dot3(v, d);
          buf->d_eps += ds * A * k.dW_de * vd;
          if (buf->mag) {
            buf->node_va[(size_t)ni * C + c] += fabs(A * k.W * ds) * norm3(d);
            buf->d_epsa += fabs(ds * A * k.dW_de * vd);
          }
          if (with_grad) {
            const double* dg = d_grad + 3 * c;
            double gd = dot3(dg, d);
            for (int a = 0; a < 3; ++a) dv[a] -= A * (k.W * dg[a] + k.Wp_r * gd * d[a]);
            double u[3];
            for (int a = 0; a < 3; ++a) u[a] = k.dW_de * v[a] + k.dWp_r_de * vd * d[a];
            buf->d_eps -= A * dot3(dg, u);
            if (buf->mag) {
              buf->node_va[(size_t)ni * C + c] +=
                  fabs(A) * (fabs(k.W) * norm3(dg) + fabs(k.Wp_r * gd) * norm3(d));
              for (int a = 0; a < 3; ++a)
                buf->d_epsa += fabs(A * dg[a]) * (fabs(k.dW_de * v[a]) + fabs(k.dWp_r_de * vd * d[a]));
            }
          }
          double* nv = buf->node_v + ((size_t)ni * C + c) * 3;
          for (int a = 0; a < 3; ++a) nv[a] += dv[a];
        } else {
          buf->node_s[(size_t)ni * C + c] += A * k.R * ds;
          buf->d_eps += ds * A * k.dR_de * t->ms[(size_t)ni * C + c];
          if (buf->mag) {
            buf->node_sa[(size_t)ni * C + c] += fabs(A * k.R * ds);
            buf->d_epsa += fabs(ds * A * k.dR_de * t->ms[(size_t)ni * C + c]);
          }
        }
      }
    } else if (t->leaf[ni]) {
      for (int32_t j = t->begin[ni]; j < t->end[ni]; ++j) {
        int64_t pi = t->order[j];
        const double* pp = t->pos + 3 * pi;
        const double* nn = t->nrm + 3 * pi;
        double dm[3] = {pp[0] - x[0], pp[1] - x[1], pp[2] - x[2]};
        double r2 = dot3(dm, dm);
        if (r2 == 0.0) continue; /* :387 */
        coeffs k = kernel_coeffs(sqrt(r2), p, 2);
        double ndot = dot3(nn, dm);
        for (int c = 0; c < C; ++c) {
          double ds = d_out[c];
          double mu = t->mu[pi * C + c];
          double A = t->ar[pi] * kInvFourPi;
          if (t->kinds[c] == 0) {
            double dmu = ds * A * k.W * ndot;
            double dn[3];
            for (int a = 0; a < 3; ++a) dn[a] = ds * A * mu * k.W * dm[a];
            buf->d_eps += ds * A * mu * k.dW_de * ndot;
            if (buf->mag) {
              buf->point_mua[pi * C + c] += fabs(dmu);
              for (int a = 0; a < 3; ++a) buf->point_na[3 * pi + a] += fabs(dn[a]);
              buf->d_epsa += fabs(ds * A * mu * k.dW_de * ndot);
            }
            if (with_grad) {
              const double* dg = d_grad + 3 * c;
              double gd = dot3(dg, dm), gn = dot3(dg, nn);
              dmu -= A * (k.W * gn + k.Wp_r * ndot * gd);
              for (int a = 0; a < 3; ++a) dn[a] -= A * mu * (k.W * dg[a] + k.Wp_r * gd * dm[a]);
              buf->d_eps -= A * mu * (k.dW_de * gn + k.dWp_r_de * ndot * gd);
              if (buf->mag) {
                buf->point_mua[pi * C + c] += fabs(A) * (fabs(k.W * gn) + fabs(k.Wp_r * ndot * gd));
                for (int a = 0; a < 3; ++a)
                  buf->point_na[3 * pi + a] += fabs(A * mu) * (fabs(k.W * dg[a]) + fabs(k.Wp_r * gd * dm[a]));
                buf->d_epsa += fabs(A * mu) * (fabs(k.dW_de * gn) + fabs(k.dWp_r_de * ndot * gd));
              }
            }
            buf->point_mu[pi * C + c] += dmu;
            for (int a = 0; a < 3; ++a) buf->point_n[3 * pi + a] += dn[a];
          } else {
            buf->point_mu[pi * C + c] += ds * A * k.R;
            buf->d_eps += ds * A * mu * k.dR_de;
            if (buf->mag) {
              buf->point_mua[pi * C + c] += fabs(ds * A * k.R);
              buf->d_epsa += fabs(ds * A * mu * k.dR_de);
            }
          }
        }
      }
    } else {
      for (int32_t c = 0; c < t->ccnt[ni]; ++c) stack[sp++] = t->cbeg[ni] + c;
    }
  }
}

/* flush_gradients: bhtree.cpp:419-463. The ancestor walk of each point is
 * independent of every other point's, so it runs over point ranges on
 * `threads` workers (the same operations per point, in the same order). */
typedef struct {
  const ora_tree* t;
  const double *node_v, *node_s;  /* summed buffers (value) or magnitudes (mag) */
  double *moments, *normals;
  int mag;
} flush_ctx;

static void flush_body(void* v, int64_t lo, int64_t hi, int w) {
  (void)w;
  flush_ctx* fc = v;
  const ora_tree* t = fc->t;
  const int C = t->C;
  for (int64_t m = lo; m < hi; ++m) { /* ancestor walk incl. the leaf, :441-457 */
    double a = t->ar[m];
    const double* n = t->nrm + 3 * m;
    for (int32_t ti = t->leaf_of[m]; ti >= 0; ti = t->parent[ti]) {
      if (!(t->area[ti] > 0)) continue;
      double f = a / t->area[ti];
      for (int c = 0; c < C; ++c) {
        if (t->kinds[c] == 0) {
          if (fc->mag) {
            /* |n . g| <= |g| for the unit normal; each normal component <= the
             * norm of its vector terms */
            double g = fc->node_v[(size_t)ti * C + c];
            fc->moments[m * C + c] += f * g;
            for (int k = 0; k < 3; ++k) fc->normals[3 * m + k] += f * fabs(t->mu[m * C + c]) * g;
          } else {
            const double* g = fc->node_v + ((size_t)ti * C + c) * 3;
            fc->moments[m * C + c] += f * dot3(n, g);
            for (int k = 0; k < 3; ++k) fc->normals[3 * m + k] += f * t->mu[m * C + c] * g[k];
          }
        } else {
          fc->moments[m * C + c] += f * fc->node_s[(size_t)ti * C + c];
        }
      }
    }
  }
}

static int flush_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void flush(const ora_tree* t, gradbuf* bufs, int nbuf, double* moments, double* normals,
                  double* d_eps) {
  const int C = t->C;
  const int64_t M = t->n;
  size_t nn = (size_t)t->nodes * C;
  double* node_v = calloc(nn * 3, sizeof(double));
  double* node_s = calloc(nn, sizeof(double));
  memset(moments, 0, (size_t)M * C * sizeof(double));
  memset(normals, 0, (size_t)M * 3 * sizeof(double));
  *d_eps = 0;
  for (int b = 0; b < nbuf; ++b) { /* :429-439 */
    for (size_t i = 0; i < nn; ++i) {
      for (int a = 0; a < 3; ++a) node_v[3 * i + a] += bufs[b].node_v[3 * i + a];
      node_s[i] += bufs[b].node_s[i];
    }
    for (size_t i = 0; i < (size_t)M * C; ++i) moments[i] += bufs[b].point_mu[i];
    for (size_t i = 0; i < (size_t)M * 3; ++i) normals[i] += bufs[b].point_n[i];
    *d_eps += bufs[b].d_eps;
  }
  flush_ctx fc = {t, node_v, node_s, moments, normals, 0};
  parallel_for(M, flush_threads(), flush_body, &fc);
  free(node_v);
  free(node_s);
}

/* the magnitude bounds through the same flush: Sum|terms| of every flushed output */
static void flush_mag(const ora_tree* t, gradbuf* bufs, int nbuf, double* mom_a, double* nrm_a,
                      double* deps_a) {
  const int C = t->C;
  const int64_t M = t->n;
  size_t nn = (size_t)t->nodes * C;
  double* va = calloc(nn, sizeof(double));
  double* sa = calloc(nn, sizeof(double));
  memset(mom_a, 0, (size_t)M * C * sizeof(double));
  memset(nrm_a, 0, (size_t)M * 3 * sizeof(double));
  *deps_a = 0;
  for (int b = 0; b < nbuf; ++b) {
    for (size_t i = 0; i < nn; ++i) va[i] += bufs[b].node_va[i], sa[i] += bufs[b].node_sa[i];
    for (size_t i = 0; i < (size_t)M * C; ++i) mom_a[i] += bufs[b].point_mua[i];
    for (size_t i = 0; i < (size_t)M * 3; ++i) nrm_a[i] += bufs[b].point_na[i];
    *deps_a += bufs[b].d_epsa;
  }
  flush_ctx fc = {t, va, sa, mom_a, nrm_a, 1};
  parallel_for(M, flush_threads(), flush_body, &fc);
  free(va);
  free(sa);
}

typedef struct {
  const ora_tree* t;
  const ora_params* p;
  double beta;
  const double *xs, *d_out, *d_grad;
  gradbuf* bufs;
} adj_ctx;

static void adjoint_body(void* v, int64_t lo, int64_t hi, int w) {
  adj_ctx* c = v;
  const int C = c->t->C;
  for (int64_t i = lo; i < hi; ++i)
    adjoint_one(c->t, c->p, c->beta, c->xs + 3 * i, c->d_out + i * C,
                c->d_grad ? c->d_grad + i * C * 3 : NULL, &c->bufs[w]);
}

void ora_adjoint_ex(const ora_tree* t, const ora_params* p, double beta, const double* xs,
                    int64_t q, const double* d_out, const double* d_grad, int threads,
                    double* moments, double* normals, double* d_eps, double* mom_abs,
                    double* nrm_abs, double* deps_abs) {
  if (threads < 1) threads = 1;
  if (threads > q) threads = q > 0 ? (int)q : 1;
  const int mag = mom_abs != NULL;
  gradbuf* bufs = xrealloc(NULL, sizeof(gradbuf) * (size_t)threads);
  for (int w = 0; w < threads; ++w) {
    if (mag)
      gradbuf_init_mag(&bufs[w], t);
    else
      gradbuf_init(&bufs[w], t);
  }
  adj_ctx c = {t, p, beta, xs, d_out, d_grad, bufs};
  parallel_for(q, threads, adjoint_body, &c);
  if (mag) flush_mag(t, bufs, threads, mom_abs, nrm_abs, deps_abs);
  flush(t, bufs, threads, moments, normals, d_eps);
  for (int w = 0; w < threads; ++w) gradbuf_free(&bufs[w]);
  free(bufs);
}

void ora_adjoint(const ora_tree* t, const ora_params* p, double beta, const double* xs, int64_t q,
                 const double* d_out, const double* d_grad, int threads, double* moments,
                 double* normals, double* d_eps) {
  ora_adjoint_ex(t, p, beta, xs, q, d_out, d_grad, threads, moments, normals, d_eps, NULL, NULL,
                 NULL);
}

/* ------------------------------------------------------------ naive sums */
/* naive_dipole_sum / naive_dipole_gradient: oracles.cpp:23-59 (Kahan). */
typedef struct {
  double sum, comp;
} kahan;
static inline void kadd(kahan* k, double v) { /* util.hpp:23-33 */
  double y = v - k->comp, s = k->sum + y;
  k->comp = (s - k->sum) - y;
  k->sum = s;
}

void ora_naive_sum(const ora_tree* t, const ora_params* p, const double* xs, int64_t q,
                   int channel, int kind, double* out, double* grad) {
  const int C = t->C;
  int singular = p->epsilon <= 0.0 && !p->desingularized;
  for (int64_t i = 0; i < q; ++i) {
    const double* x = xs + 3 * i;
    kahan s = {0, 0}, gx = {0, 0}, gy = {0, 0}, gz = {0, 0};
    for (int64_t m = 0; m < t->n; ++m) {
      const double* pp = t->pos + 3 * m;
      const double* nn = t->nrm + 3 * m;
      double d[3] = {pp[0] - x[0], pp[1] - x[1], pp[2] - x[2]};
      double r2 = dot3(d, d);
      if (r2 == 0.0 && singular) continue;
      double w, g[3] = {0, 0, 0};
      if (kind == 0) { /* regularized_poisson / grad (kernels.cpp:163-182) */
        if (r2 == 0.0 && !p->desingularized) {
          w = p->coincident_value;
        } else {
          coeffs k = kernel_coeffs(sqrt(r2), p, 2);
          double nd = dot3(nn, d);
          w = kInvFourPi * k.W * nd;
          for (int a = 0; a < 3; ++a) g[a] = -kInvFourPi * (k.W * nn[a] + k.Wp_r * nd * d[a]);
        }
      } else { /* radial_regularized (kernels.cpp:184-190) */
        if (r2 == 0.0 && !p->desingularized) {
          w = 0.0;
        } else {
          coeffs k = kernel_coeffs(sqrt(r2), p, 2);
          w = kInvFourPi * k.R;
          for (int a = 0; a < 3; ++a) g[a] = -kInvFourPi * k.Rp_r * d[a];
        }
      }
      double sc = t->ar[m] * t->mu[m * C + channel];
      kadd(&s, sc * w);
      kadd(&gx, sc * g[0]), kadd(&gy, sc * g[1]), kadd(&gz, sc * g[2]);
    }
    out[i] = s.sum;
    if (grad) grad[3 * i] = gx.sum, grad[3 * i + 1] = gy.sum, grad[3 * i + 2] = gz.sum;
  }
}

/* naive_adjoint: oracles.cpp:61-105 */
void ora_naive_adjoint(const ora_tree* t, const ora_params* p, const double* xs, int64_t q,
                       const double* d_out, const double* d_grad, double* moments,
                       double* normals, double* d_eps) {
  const int C = t->C;
  memset(moments, 0, sizeof(double) * (size_t)t->n * C);
  memset(normals, 0, sizeof(double) * (size_t)t->n * 3);
  *d_eps = 0;
  for (int64_t i = 0; i < q; ++i) {
    const double* x = xs + 3 * i;
    for (int64_t m = 0; m < t->n; ++m) {
      const double* pp = t->pos + 3 * m;
      const double* nn = t->nrm + 3 * m;
      double d[3] = {pp[0] - x[0], pp[1] - x[1], pp[2] - x[2]};
      double r2 = dot3(d, d);
      if (r2 == 0.0) continue;
      coeffs k = kernel_coeffs(sqrt(r2), p, 2);
      double ndot = dot3(nn, d), A = t->ar[m] * kInvFourPi;
      for (int c = 0; c < C; ++c) {
        double ds = d_out[i * C + c], mu = t->mu[m * C + c];
        if (t->kinds[c] == 0) {
          moments[m * C + c] += ds * A * k.W * ndot;
          for (int a = 0; a < 3; ++a) normals[3 * m + a] += ds * A * mu * k.W * d[a];
          *d_eps += ds * A * mu * k.dW_de * ndot;
          if (d_grad) {
            const double* dg = d_grad + (i * C + c) * 3;
            double gd = dot3(dg, d), gn = dot3(dg, nn);
            moments[m * C + c] -= A * (k.W * gn + k.Wp_r * ndot * gd);
            for (int a = 0; a < 3; ++a) normals[3 * m + a] -= A * mu * (k.W * dg[a] + k.Wp_r * gd * d[a]);
            *d_eps -= A * mu * (k.dW_de * gn + k.dWp_r_de * ndot * gd);
          }
        } else {
          moments[m * C + c] += ds * A * k.R;
          *d_eps += ds * A * mu * k.dR_de;
        }
      }
    }
  }
}

/* ------------------------------------------------------------ render step */
/* splitmix64-based counter RNG shared with the CUDA sampler (render.cu). */
double ora_uniform(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53;
}

/* Stratified samples in RaySamples form (renderer.hpp:322-326):
 * t_j = t_near + span * ((j + u_j) / S), delta_0 = t_0 - t_near,
 * delta_j = t_j - t_{j-1} (as sample_ray computes deltas, renderer.cpp:82-84). */
void ora_stratified_samples(int64_t R, int32_t S, double t_near, double t_far, uint64_t seed,
                            int64_t ray_offset, double* ts, double* deltas) {
  double span = t_far - t_near;
  for (int64_t r = 0; r < R; ++r)
    for (int32_t j = 0; j < S; ++j) {
      uint64_t ctr = (uint64_t)(ray_offset + r) * (uint64_t)S + (uint64_t)j;
      double u = ora_uniform(seed, ctr);
      double tj = t_near + span * (((double)j + u) / (double)S);
      ts[r * S + j] = tj;
      deltas[r * S + j] = tj - (j == 0 ? t_near : ts[r * S + j - 1]);
    }
}

/* logistic: radiance.cpp:30-38 */
static double logistic(double x) {
  if (x >= 0) {
    double e = exp(-x);
    return 1.0 / (1.0 + e);
  }
  double e = exp(x);
  return e / (1.0 + e);
}

typedef struct {
  const ora_tree* t;
  const ora_params* p;
  double beta, lambda;
  const double *bg, *rays, *ts, *deltas, *target;
  double scale;
  int32_t S;
  double* rgb;
  gradbuf* bufs;
  double *d_lambda, *d_bg; /* per worker */
} render_ctx;

/* render_ray (renderer.cpp:106-171, no lights) + render_ray_backward
 * (:173-231) with the direct-rgb head (radiance.cpp:133-145, 160-174). */
static void render_body(void* v, int64_t lo, int64_t hi, int w) {
  render_ctx* c = v;
  const ora_tree* t = c->t;
  const int C = t->C, S = c->S;
  const double lam = c->lambda;
  double* out = xrealloc(NULL, sizeof(double) * C);
  double* grad = xrealloc(NULL, sizeof(double) * C * 3);
  double* d_out = xrealloc(NULL, sizeof(double) * C);
  double* d_grad = xrealloc(NULL, sizeof(double) * C * 3);
  /* tape per sample: x(3) f gradf(3) s trans p rgb(3) */
  double* tape = xrealloc(NULL, sizeof(double) * 13 * (size_t)S);
  double* dp = xrealloc(NULL, sizeof(double) * S);
  double* dsig = xrealloc(NULL, sizeof(double) * S);
  for (int64_t r = lo; r < hi; ++r) {
    const double* o = c->rays + 6 * r;
    const double* dir = o + 3;
    const double* ts = c->ts + r * S;
    const double* dl = c->deltas + r * S;
    double trans = 1.0, rgb[3] = {0, 0, 0};
    for (int j = 0; j < S; ++j) {
      double* tp = tape + 13 * j;
      double x[3] = {o[0] + ts[j] * dir[0], o[1] + ts[j] * dir[1], o[2] + ts[j] * dir[2]};
      primal_one(t, c->p, c->beta, x, 1, 0, out, grad, NULL);
      double f = 0.5 - out[0];
      double gf[3] = {-grad[0], -grad[1], -grad[2]};
      double s = dot3(dir, gf);
      double sigma = lam * ora_normal_hazard(lam * f) * fabs(s); /* sigma_of, :100-102 */
      double hr[3];
      for (int k = 0; k < 3; ++k) hr[k] = logistic(out[1 + k]);
      double E = exp(-sigma * dl[j]);
      double pj = trans * (1.0 - E);
      for (int k = 0; k < 3; ++k) rgb[k] += pj * hr[k];
      memcpy(tp, x, sizeof x);
      tp[3] = f;
      memcpy(tp + 4, gf, sizeof gf);
      tp[7] = s, tp[8] = trans, tp[9] = pj;
      memcpy(tp + 10, hr, sizeof hr);
      trans *= E;
    }
    double res[3];
    for (int k = 0; k < 3; ++k) res[k] = rgb[k] + trans * c->bg[k];
    memcpy(c->rgb + 3 * r, res, sizeof res);
    /* L2 loss gradient supplied by the harness */
    double drgb[3];
    for (int k = 0; k < 3; ++k) drgb[k] = c->scale * (res[k] - c->target[3 * r + k]);
    double sum_p = 0;
    for (int j = 0; j < S; ++j) {
      const double* tp = tape + 13 * j;
      double rd[3] = {tp[10] - c->bg[0], tp[11] - c->bg[1], tp[12] - c->bg[2]};
      dp[j] = dot3(drgb, rd);
      sum_p += tp[9];
    }
    for (int k = 0; k < 3; ++k) c->d_bg[3 * w + k] += (1.0 - sum_p) * drgb[k];
    double suffix = 0;
    for (int j = S; j-- > 0;) {
      const double* tp = tape + 13 * j;
      double E = tp[8] > 0 ? 1.0 - tp[9] / tp[8] : 0.0;
      dsig[j] = dl[j] * (tp[8] * E * dp[j] - suffix);
      suffix += tp[9] * dp[j];
    }
    for (int j = 0; j < S; ++j) {
      const double* tp = tape + 13 * j;
      double drad[3] = {tp[9] * drgb[0], tp[9] * drgb[1], tp[9] * drgb[2]};
      double dgf[3] = {0, 0, 0}; /* direct-rgb head has no normal input */
      double u = lam * tp[3];
      double haz = ora_normal_hazard(u);
      double dhaz = -u * haz - haz * haz;
      double abs_s = fabs(tp[7]);
      double sgn_s = tp[7] > 0 ? 1.0 : (tp[7] < 0 ? -1.0 : 0.0);
      double d_f = dsig[j] * lam * lam * abs_s * dhaz;
      c->d_lambda[w] += dsig[j] * (haz * abs_s + lam * abs_s * dhaz * tp[3]);
      for (int k = 0; k < 3; ++k) dgf[k] += dsig[j] * lam * haz * sgn_s * dir[k];
      memset(d_out, 0, sizeof(double) * C);
      memset(d_grad, 0, sizeof(double) * C * 3);
      d_out[0] = -d_f;
      for (int k = 0; k < 3; ++k) d_grad[k] = -dgf[k];
      for (int k = 0; k < 3; ++k) /* logistic backward, radiance.cpp:166 */
        d_out[1 + k] = drad[k] * tp[10 + k] * (1.0 - tp[10 + k]);
      adjoint_one(t, c->p, c->beta, tp, d_out, d_grad, &c->bufs[w]);
    }
  }
  free(out), free(grad), free(d_out), free(d_grad), free(tape), free(dp), free(dsig);
}

void ora_render_step_ex(const ora_tree* t, const ora_params* p, double beta, double lambda,
                        const double* background, const double* rays, int64_t R, int32_t S,
                        const double* ts, const double* deltas, const double* target,
                        double scale, int threads, double* rgb, double* moments, double* normals,
                        double* d_eps, double* d_lambda, double* d_bg, double* mom_abs,
                        double* nrm_abs, double* deps_abs) {
  if (threads < 1) threads = 1;
  if (threads > R) threads = R > 0 ? (int)R : 1;
  const int mag = mom_abs != NULL;
  gradbuf* bufs = xrealloc(NULL, sizeof(gradbuf) * (size_t)threads);
  double* dl = calloc((size_t)threads, sizeof(double));
  double* db = calloc((size_t)threads * 3, sizeof(double));
  for (int w = 0; w < threads; ++w) {
    if (mag)
      gradbuf_init_mag(&bufs[w], t);
    else
      gradbuf_init(&bufs[w], t);
  }
  render_ctx c = {t, p, beta, lambda, background, rays, ts, deltas, target, scale, S,
                  rgb, bufs, dl, db};
  parallel_for(R, threads, render_body, &c);
  if (mag) flush_mag(t, bufs, threads, mom_abs, nrm_abs, deps_abs);
  flush(t, bufs, threads, moments, normals, d_eps);
  *d_lambda = 0;
  d_bg[0] = d_bg[1] = d_bg[2] = 0;
  for (int w = 0; w < threads; ++w) {
    *d_lambda += dl[w];
    for (int k = 0; k < 3; ++k) d_bg[k] += db[3 * w + k];
    gradbuf_free(&bufs[w]);
  }
  free(bufs), free(dl), free(db);
}

void ora_render_step(const ora_tree* t, const ora_params* p, double beta, double lambda,
                     const double* background, const double* rays, int64_t R, int32_t S,
                     const double* ts, const double* deltas, const double* target, double scale,
                     int threads, double* rgb, double* moments, double* normals, double* d_eps,
                     double* d_lambda, double* d_bg) {
  ora_render_step_ex(t, p, beta, lambda, background, rays, R, S, ts, deltas, target, scale,
                     threads, rgb, moments, normals, d_eps, d_lambda, d_bg, NULL, NULL, NULL);
}

/* ------------------------------------------------------- mean kNN spacing */
/* OrientedPointCloud::mean_knn_spacing (pointcloud.cpp:51-65): for every point
 * the k nearest OTHER points (the k+1 nearest including itself, minus the
 * first), distances summed in ascending order. Exact kNN over a uniform grid
 * instead of the reference's kd-tree (kdtree.hpp) — same neighbour sets. */
typedef struct {
  double lo[3], cell;
  int64_t dim[3];
  int64_t *start, *idx;
} grid3;

static int64_t gclamp(int64_t v, int64_t n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); }

double ora_mean_knn_spacing(const double* pos, int64_t n, int k) {
  if (n < 2) return 0.0;
  int kk = k + 1 < n ? k + 1 : (int)n;
  grid3 g;
  double hi[3];
  for (int a = 0; a < 3; ++a) g.lo[a] = hi[a] = pos[a];
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      if (pos[3 * i + a] < g.lo[a]) g.lo[a] = pos[3 * i + a];
      if (pos[3 * i + a] > hi[a]) hi[a] = pos[3 * i + a];
    }
  double ext = 0;
  for (int a = 0; a < 3; ++a) ext = fmax(ext, hi[a] - g.lo[a]);
  if (ext <= 0) ext = 1;
  double target_cells = (double)n / 4.0;
  g.cell = ext / cbrt(target_cells);
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) {
    g.dim[a] = (int64_t)((hi[a] - g.lo[a]) / g.cell) + 1;
    total *= g.dim[a];
  }
  g.start = calloc((size_t)total + 1, sizeof(int64_t));
  g.idx = xrealloc(NULL, sizeof(int64_t) * (size_t)n);
  int64_t* cellof = xrealloc(NULL, sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t c[3];
    for (int a = 0; a < 3; ++a) c[a] = gclamp((int64_t)((pos[3 * i + a] - g.lo[a]) / g.cell), g.dim[a]);
    cellof[i] = (c[2] * g.dim[1] + c[1]) * g.dim[0] + c[0];
    g.start[cellof[i] + 1]++;
  }
  for (int64_t c = 0; c < total; ++c) g.start[c + 1] += g.start[c];
  int64_t* fill = xrealloc(NULL, sizeof(int64_t) * (size_t)total);
  memcpy(fill, g.start, sizeof(int64_t) * (size_t)total);
  for (int64_t i = 0; i < n; ++i) g.idx[fill[cellof[i]]++] = i;
  free(fill);
  double* best = xrealloc(NULL, sizeof(double) * (size_t)kk); /* ascending squared dists */
  double sum = 0.0;
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* q = pos + 3 * i;
    int nb = 0;
    int64_t c0[3];
    for (int a = 0; a < 3; ++a) c0[a] = gclamp((int64_t)((q[a] - g.lo[a]) / g.cell), g.dim[a]);
    for (int64_t ring = 0;; ++ring) {
      for (int64_t z = c0[2] - ring; z <= c0[2] + ring; ++z)
        for (int64_t y = c0[1] - ring; y <= c0[1] + ring; ++y)
          for (int64_t x = c0[0] - ring; x <= c0[0] + ring; ++x) {
            if (z < 0 || y < 0 || x < 0 || z >= g.dim[2] || y >= g.dim[1] || x >= g.dim[0]) continue;
            int64_t dz = z - c0[2], dy = y - c0[1], dx = x - c0[0];
            if (llabs(dz) != ring && llabs(dy) != ring && llabs(dx) != ring) continue;
            int64_t cell = (z * g.dim[1] + y) * g.dim[0] + x;
            for (int64_t s = g.start[cell]; s < g.start[cell + 1]; ++s) {
              const double* pp = pos + 3 * g.idx[s];
              double d[3] = {pp[0] - q[0], pp[1] - q[1], pp[2] - q[2]};
              double d2 = dot3(d, d);
              if (nb < kk || d2 < best[nb - 1]) {
                int w = nb < kk ? nb++ : kk - 1;
                while (w > 0 && best[w - 1] > d2) best[w] = best[w - 1], --w;
                best[w] = d2;
              }
            }
          }
      /* every unvisited point is at least ring * cell away (per axis) */
      double reach = (double)ring * g.cell;
      int covered = c0[0] - ring <= 0 && c0[1] - ring <= 0 && c0[2] - ring <= 0 &&
                    c0[0] + ring >= g.dim[0] - 1 && c0[1] + ring >= g.dim[1] - 1 &&
                    c0[2] + ring >= g.dim[2] - 1;
      if ((nb == kk && best[kk - 1] <= reach * reach) || covered) break;
    }
    for (int j = 1; j < nb; ++j) {
      sum += sqrt(best[j]);
      ++count;
    }
  }
  free(best), free(g.start), free(g.idx), free(cellof);
  return count ? sum / (double)count : 0.0;
}

/* ------------------------------------------------------------------ Adam */
/* Adam::step: optimizer.cpp:65-81 */
void ora_adam_step(double* params, const double* grads, double* m, double* v, int64_t n,
                   double lr, double beta1, double beta2, double eps, int64_t t) {
  double c1 = 1.0 - pow(beta1, (double)t);
  double c2 = 1.0 - pow(beta2, (double)t);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + (1.0 - beta1) * grads[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * grads[i] * grads[i];
    params[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}

/* ------------------------------------------------------- query generators */
/* sample_grid: meshing.cpp:33-59. geometry_field(x) = 0.5 - primal_channel(x,
 * 0) (fields.cpp:27-29); node (i, j, k) = lo + f .* (hi - lo) with f = i /
 * (dims - 1) (FieldGrid::node, meshing.cpp:25-30). If |hi - lo| == 0 the box
 * is the bounding box of pos (pointcloud.cpp:22-29) padded by 5% (:38-43). */
int ora_sample_grid(const ora_tree* t, const ora_params* p, double beta, const int32_t* res,
                    const double* lo_in, const double* hi_in, const double* pos, int64_t n,
                    int threads, double* values, double* lo_out, double* hi_out) {
  for (int a = 0; a < 3; ++a)
    if (res[a] < 2) return 2; /* DataError */
  double lo[3] = {lo_in[0], lo_in[1], lo_in[2]}, hi[3] = {hi_in[0], hi_in[1], hi_in[2]};
  double d[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  if (sqrt(dot3(d, d)) == 0.0) {
    for (int a = 0; a < 3; ++a) lo[a] = INFINITY, hi[a] = -INFINITY;
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        double v = pos[3 * i + a];
        lo[a] = v < lo[a] ? v : lo[a]; /* cwiseMin */
        hi[a] = hi[a] < v ? v : hi[a]; /* cwiseMax */
      }
    for (int a = 0; a < 3; ++a) {
      double pad = 0.05 * (hi[a] - lo[a]);
      lo[a] -= pad;
      hi[a] += pad;
    }
  }
  int64_t total = (int64_t)res[0] * res[1] * res[2];
  double* xs = malloc((size_t)total * 3 * sizeof(double));
  for (int64_t g = 0; g < total; ++g) {
    int64_t i = g % res[0], j = (g / res[0]) % res[1], k = g / ((int64_t)res[0] * res[1]);
    double f[3] = {(double)i / (res[0] - 1), (double)j / (res[1] - 1), (double)k / (res[2] - 1)};
    for (int a = 0; a < 3; ++a) xs[3 * g + a] = lo[a] + f[a] * (hi[a] - lo[a]);
  }
  ora_primal(t, p, beta, xs, total, 2, 0, values, NULL, NULL, threads);
  for (int64_t g = 0; g < total; ++g) values[g] = 0.5 - values[g];
  free(xs);
  for (int a = 0; a < 3; ++a) lo_out[a] = lo[a], hi_out[a] = hi[a];
  return 0;
}

/* sample_ray: renderer.cpp:46-86 (probe pass, first sign change of f, then
 * sparse / dense / sparse or uniform samples; delta[j] = t[j] - t[j-1]). */
typedef struct {
  const ora_tree* t;
  const ora_params* p;
  double beta;
  const double* rays;
  double t_near, t_far;
  const int32_t* cnt5; /* probe, sparse_before, dense_at, sparse_after, uniform */
  int32_t max_s;
  double *ts, *delta;
  int32_t* count;
  uint8_t* bracketed;
} ray_ctx;

static void ray_body(void* v, int64_t lo_r, int64_t hi_r, int w) {
  (void)w;
  ray_ctx* c = v;
  for (int64_t r = lo_r; r < hi_r; ++r) {
    const double* ray = c->rays + 6 * r;
    double* t = c->ts + r * c->max_s;
    double* dl = c->delta + r * c->max_s;
    double span = c->t_far - c->t_near;
    int m = 0, br = 0;
    if (span < 1e-9) {
      t[0] = 0.5 * (c->t_near + c->t_far);
      dl[0] = t[0] - c->t_near;
      c->count[r] = 1;
      c->bracketed[r] = 0;
      continue;
    }
    int n = c->cnt5[0] < 2 ? 2 : c->cnt5[0];
    double prev_f = 0, prev_t = 0, blo = 0, bhi = 0;
    for (int i = 0; i < n; ++i) {
      double tt = c->t_near + span * i / (n - 1);
      double x[3] = {ray[0] + tt * ray[3], ray[1] + tt * ray[4], ray[2] + tt * ray[5]};
      double v0;
      primal_one(c->t, c->p, c->beta, x, 2, 0, &v0, NULL, NULL);
      double f = 0.5 - v0;
      if (i > 0 && ((prev_f > 0 && f <= 0) || (prev_f <= 0 && f > 0))) {
        br = 1;
        blo = prev_t;
        bhi = tt;
        break;
      }
      prev_f = f;
      prev_t = tt;
    }
#define EMIT(L, H, K)                                                     \
  do {                                                                    \
    double lo_ = (L), hi_ = (H);                                          \
    int k_ = (K);                                                         \
    for (int i_ = 0; i_ < k_ && m < c->max_s; ++i_)                       \
      t[m++] = lo_ + (hi_ - lo_) * (i_ + 0.5) / k_;                        \
  } while (0)
    if (!br) {
      EMIT(c->t_near, c->t_far, c->cnt5[4] > 1 ? c->cnt5[4] : 1);
    } else {
      EMIT(c->t_near, blo, c->cnt5[1]);
      EMIT(blo, bhi, c->cnt5[2] > 1 ? c->cnt5[2] : 1);
      EMIT(bhi, c->t_far, c->cnt5[3]);
    }
#undef EMIT
    for (int j = 0; j < m; ++j) dl[j] = t[j] - (j == 0 ? c->t_near : t[j - 1]);
    c->count[r] = m;
    c->bracketed[r] = (uint8_t)br;
  }
}

void ora_sample_rays(const ora_tree* t, const ora_params* p, double beta, const double* rays,
                     int64_t R, double t_near, double t_far, const int32_t* counts5,
                     int32_t max_s, int threads, double* ts, double* delta, int32_t* count,
                     uint8_t* bracketed) {
  ray_ctx c = {t, p, beta, rays, t_near, t_far, counts5, max_s, ts, delta, count, bracketed};
  parallel_for(R, threads, ray_body, &c);
}
