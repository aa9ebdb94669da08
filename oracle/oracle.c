/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
 *
 * A plain-C restatement of the arithmetic of the reference package
 * `adacluster` 0.1.0 (/root/reference/pkg/src/adacluster) on its hot path,
 * written so that every reduction happens in the order numpy 2.3 /
 * OpenBLAS 0.3.30 (SkylakeX) performs it in the container where the
 * reference was run (re-measured by
 * oracle/probe_blas.py).  Results are bit-identical to the reference for
 * clustering, selection and TensorQuest; attention is computed in the
 * reference's f32 formulation by oracle.py with numpy (tolerance-checked).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  Built by oracle/Makefile into oracle/_build/.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---- row-parallel helper: rows are independent, so splitting them across
 * threads leaves every value bit-identical ----------------------------- */
typedef void (*row_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { row_fn fn; void* ctx; int64_t lo, hi; } par_job;
static int g_threads = 0;
int oc_num_threads(void) {
  if (g_threads <= 0) {
    const char* e = getenv("ORACLE_THREADS");
    long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    g_threads = (int)(t < 1 ? 1 : (t > 256 ? 256 : t));
  }
  return g_threads;
}
void oc_set_threads(int t) { g_threads = t; }
static void* par_entry(void* p) {
  par_job* j = (par_job*)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static void par_rows(int64_t n, row_fn fn, void* ctx) {
  int T = oc_num_threads();
  if (n < 4096 || T == 1) { fn(ctx, 0, n); return; }
  if (T > 256) T = 256;
  pthread_t th[256];
  par_job jobs[256];
  const int64_t per = (n + T - 1) / T;
  int used = 0;
  for (int t = 0; t < T; ++t) {
    const int64_t lo = t * per, hi = lo + per < n ? lo + per : n;
    if (lo >= hi) break;
    jobs[t] = (par_job){fn, ctx, lo, hi};
    ++used;
  }
  for (int t = 1; t < used; ++t) pthread_create(&th[t], NULL, par_entry, &jobs[t]);
  par_entry(&jobs[0]);
  for (int t = 1; t < used; ++t) pthread_join(th[t], NULL);
}

#define ORD_SEQ 0
#define ORD_L16 1
#define ORD_GEMV8 2

/* ---- numpy pairwise summation (loops_utils.h.src: pairwise_sum) -------- */
static float pw_leaf_f(const float* a, int64_t n, int64_t s) {
  if (n < 8) {
    float r = 0.f;
    for (int64_t i = 0; i < n; ++i) r = r + a[i * s];
    return r;
  }
  float r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j * s];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + a[(i + j) * s];
  float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + a[i * s];
  return res;
}
static float pw_f_s(const float* a, int64_t n, int64_t s) {
  if (n <= 128) return pw_leaf_f(a, n, s);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_f_s(a, n2, s) + pw_f_s(a + n2 * s, n - n2, s);
}
static double pw_leaf_d(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = r + a[i];
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + a[i];
  return res;
}
static double pw_d(const double* a, int64_t n) {
  if (n <= 128) return pw_leaf_d(a, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_d(a, n2) + pw_d(a + n2, n - n2);
}

float oc_pw_f32(const float* a, int64_t n) { return pw_f_s(a, n, 1); }
double oc_pw_f64(const double* a, int64_t n) { return pw_d(a, n); }

/* float(arr.mean()) for an f32 array: f32(f64(pairwise_sum) / n) */
static float mean_f32(const float* a, int64_t n) {
  return (float)((double)pw_f_s(a, n, 1) / (double)n);
}

/* ---- row reductions over D ------------------------------------------- */
static float rowsq(const float* x, int d, float* tmp) {
  for (int t = 0; t < d; ++t) tmp[t] = x[t] * x[t];
  return pw_f_s(tmp, d, 1);
}
void oc_rowsq(const float* x, int64_t n, int d, float* out) {
  float* tmp = (float*)malloc(sizeof(float) * d);
  for (int64_t i = 0; i < n; ++i) out[i] = rowsq(x + i * d, d, tmp);
  free(tmp);
}

/* tensorops.py:59-76 */
void oc_l2norm(const float* x, int64_t n, int d, float* out, uint8_t* degen) {
  float* tmp = (float*)malloc(sizeof(float) * d);
  for (int64_t i = 0; i < n; ++i) {
    const float nrm = sqrtf(rowsq(x + i * d, d, tmp));
    const int dg = nrm < 1e-12f;
    const int unit = fabsf(nrm - 1.0f) <= 2e-6f;
    const float safe = (dg || unit) ? 1.0f : nrm;
    for (int t = 0; t < d; ++t) out[i * d + t] = dg ? 0.f : x[i * d + t] / safe;
    degen[i] = (uint8_t)dg;
  }
  free(tmp);
}

/* ---- OpenBLAS order of f32 x @ c.T ------------------------------------ */
int oc_gemm_order(int64_t m, int64_t n, int64_t d) {
  if (m == 1 || n == 1) return ORD_GEMV8;
  if (m * n <= 1200 && d >= 32) return ORD_L16;
  return ORD_SEQ;
}

static float dot_ord(const float* x, const float* c, int d, int order, int halves) {
  if (order == ORD_L16) {
    float r[16] = {0};
    for (int t = 0; t < d; ++t) r[t & 15] = fmaf(x[t], c[t], r[t & 15]);
    float s[8], u[4];
    if (halves) {
      for (int l = 0; l < 8; ++l) s[l] = r[l] + r[l + 8];
      for (int l = 0; l < 4; ++l) u[l] = s[l] + s[l + 4];
      return (u[0] + u[2]) + (u[1] + u[3]);
    }
    for (int l = 0; l < 8; ++l) s[l] = r[2 * l] + r[2 * l + 1];
    for (int l = 0; l < 4; ++l) u[l] = s[2 * l] + s[2 * l + 1];
    return (u[0] + u[1]) + (u[2] + u[3]);
  }
  if (order == ORD_GEMV8) {
    float a[8] = {0};
    for (int t = 0; t < d; ++t) a[t & 7] = fmaf(x[t], c[t], a[t & 7]);
    const float s0 = a[0] + a[4], s1 = a[1] + a[5], s2 = a[2] + a[6], s3 = a[3] + a[7];
    return (s0 + s1) + (s2 + s3);
  }
  float acc = 0.f;
  for (int t = 0; t < d; ++t) acc = fmaf(x[t], c[t], acc);
  return acc;
}

/* out[i*n+j] = a[i] . b[j] in the reference's order for an (m, n, d) call */
void oc_matmul_nt(const float* a, int64_t m, const float* b, int64_t n, int d, float* out) {
  const int order = oc_gemm_order(m, n, d);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int hv = (i >= m - m % 4) && (j >= n - n % 4);
      out[i * n + j] = dot_ord(a + i * d, b + j * d, d, order, hv);
    }
}

static float np_max(float a, float b) { return (a >= b || isnan(a)) ? a : b; }
static float np_min(float a, float b) { return (a <= b || isnan(a)) ? a : b; }

/* clustering.py:68-75 + :94-97.  labels/best (assigned squared distance);
 * dfull optional [n, k].  `order` < 0 selects the reference's dispatch. */
typedef struct {
  const float *x, *c, *cc;
  int64_t n;
  int d, k, order;
  int32_t* labels;
  float *best, *dfull;
} assign_ctx;

static void assign_rows(void* p, int64_t lo, int64_t hi) {
  const assign_ctx* a = (const assign_ctx*)p;
  const int d = a->d, k = a->k;
  const int64_t n = a->n;
  float* tmp = (float*)malloc(sizeof(float) * d);
  for (int64_t i = lo; i < hi; ++i) {
    const float* xr = a->x + i * d;
    const float xx = rowsq(xr, d, tmp);
    float bd = INFINITY;
    int bl = -1;
    for (int j = 0; j < k; ++j) {
      const int hv = (i >= n - n % 4) && (j >= k - k % 4);
      const float xc = dot_ord(xr, a->c + (int64_t)j * d, d, a->order, hv);
      float dd = (xx - 2.0f * xc) + a->cc[j];
      dd = np_max(dd, 0.f);
      if (a->dfull) a->dfull[i * k + j] = dd;
      if (bl < 0 || dd < bd) { bd = dd; bl = j; }
    }
    a->labels[i] = bl;
    a->best[i] = bd;
  }
  free(tmp);
}

void oc_assign(const float* x, int64_t n, int d, const float* c, int k, int order,
               int32_t* labels, float* best, float* dfull) {
  if (order < 0) order = oc_gemm_order(n, k, d);
  float* tmp = (float*)malloc(sizeof(float) * d);
  float* cc = (float*)malloc(sizeof(float) * (k > 0 ? k : 1));
  for (int j = 0; j < k; ++j) cc[j] = rowsq(c + (int64_t)j * d, d, tmp);
  free(tmp);
  assign_ctx a = {x, c, cc, n, d, k, order, labels, best, dfull};
  par_rows(n, assign_rows, &a);
  free(cc);
}

/* clustering.py:100-116 on the assigned distances.  Returns repairs done. */
static int repair_empty(const float* x, int64_t n, int d, float* centers, int k,
                        int32_t* labels, float* best, int64_t* counts) {
  int repairs = 0;
  for (int guard = 0; guard < k; ++guard) {
    memset(counts, 0, sizeof(int64_t) * k);
    for (int64_t i = 0; i < n; ++i) counts[labels[i]]++;
    int c = -1;
    for (int j = 0; j < k; ++j)
      if (counts[j] == 0) { c = j; break; }
    if (c < 0) return repairs;
    int64_t far = 0;
    for (int64_t i = 1; i < n; ++i)
      if (best[i] > best[far]) far = i;
    memcpy(centers + (int64_t)c * d, x + far * d, sizeof(float) * d);
    labels[far] = c;
    best[far] = 0.f;
    ++repairs;
  }
  memset(counts, 0, sizeof(int64_t) * k);
  for (int64_t i = 0; i < n; ++i) counts[labels[i]]++;
  return repairs;
}

/* f64 mean of members in member order (np.add.reduceat / np.add.at) */
void oc_segment_mean(const float* x, int64_t n, int d, const int32_t* labels, int k,
                     float* out) {
  int64_t* counts = (int64_t*)calloc(k > 0 ? k : 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) counts[labels[i]]++;
  double* acc = (double*)calloc((size_t)k * d, sizeof(double));
  int64_t* seen = (int64_t*)calloc(k > 0 ? k : 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    const int j = labels[i];
    double* a = acc + (int64_t)j * d;
    if (seen[j]++ == 0)
      for (int t = 0; t < d; ++t) a[t] = (double)x[i * d + t];
    else
      for (int t = 0; t < d; ++t) a[t] = a[t] + (double)x[i * d + t];
  }
  for (int j = 0; j < k; ++j)
    for (int t = 0; t < d; ++t)
      out[(int64_t)j * d + t] = (float)(acc[(int64_t)j * d + t] / (double)counts[j]);
  free(seen);
  free(acc);
  free(counts);
}

/* clustering.py:119-152.  centers in/out [k, d]; inertia [max_iter].
 * Returns the number of Lloyd iterations executed. */
int oc_lloyd(const float* x, int64_t n, int d, float* centers, int k, int max_iter, double tol,
             int32_t* labels, float* best, int64_t* counts, float* inertia, int* repairs_out) {
  const int order = oc_gemm_order(n, k, d);
  float* newc = (float*)malloc(sizeof(float) * (size_t)k * d);
  float* mv = (float*)malloc(sizeof(float) * (k > 0 ? k : 1));
  float* tmp = (float*)malloc(sizeof(float) * d);
  int n_iter = 0, repairs = 0;
  for (int it = 0; it < max_iter; ++it) {
    ++n_iter;
    oc_assign(x, n, d, centers, k, order, labels, best, NULL);
    repairs += repair_empty(x, n, d, centers, k, labels, best, counts);
    inertia[it] = pw_f_s(best, n, 1);
    oc_segment_mean(x, n, d, labels, k, newc);
    for (int j = 0; j < k; ++j) {
      for (int t = 0; t < d; ++t) {
        const float df = newc[(int64_t)j * d + t] - centers[(int64_t)j * d + t];
        tmp[t] = df * df;
      }
      mv[j] = sqrtf(pw_f_s(tmp, d, 1));
    }
    const float movement = mean_f32(mv, k);
    memcpy(centers, newc, sizeof(float) * (size_t)k * d);
    if ((double)movement < tol) break;
  }
  oc_assign(x, n, d, centers, k, order, labels, best, NULL);
  repairs += repair_empty(x, n, d, centers, k, labels, best, counts);
  if (repairs_out) *repairs_out = repairs;
  free(tmp);
  free(mv);
  free(newc);
  return n_iter;
}

typedef struct {
  const float* x;
  const float* c;
  float* closest;
  int d, init;
} kpp_ctx;

/* closest = min(closest, ((x - c) ** 2).sum(axis=1)) over a row range */
static void kpp_rows(void* p, int64_t lo, int64_t hi) {
  const kpp_ctx* a = (const kpp_ctx*)p;
  const int d = a->d;
  float* tmp = (float*)malloc(sizeof(float) * d);
  for (int64_t i = lo; i < hi; ++i) {
    for (int t = 0; t < d; ++t) {
      const float df = a->x[i * d + t] - a->c[t];
      tmp[t] = df * df;
    }
    const float v = pw_f_s(tmp, d, 1);
    a->closest[i] = a->init ? v : np_min(a->closest[i], v);
  }
  free(tmp);
}

/* clustering.py:78-91.  draws[0] = first index, draws[i] = u_i or -(idx+1)
 * (forced rng.integers result).  Returns -1, or the step i at which
 * `total <= 0` was met with an unforced draw (centres [0, i) are valid). */
int oc_kmeanspp(const float* x, int64_t n, int d, int k, const double* draws, float* centers) {
  float* closest = (float*)malloc(sizeof(float) * n);
  float* tmp = (float*)malloc(sizeof(float) * d);
  double* cdf = (double*)malloc(sizeof(double) * n);
  int64_t idx = (int64_t)draws[0];
  memcpy(centers, x + idx * d, sizeof(float) * d);
  kpp_ctx kc = {x, centers, closest, d, 1};
  par_rows(n, kpp_rows, &kc);
  int stop = -1;
  for (int s = 1; s < k; ++s) {
    const float total = pw_f_s(closest, n, 1);
    if (total <= 0.f) {
      if (draws[s] >= 0) { stop = s; break; }
      idx = (int64_t)(-draws[s]) - 1;
    } else {
      double run = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        run = run + (double)(closest[i] / total);
        cdf[i] = run;
      }
      const double last = cdf[n - 1];
      const double u = draws[s];
      idx = n;
      for (int64_t i = 0; i < n; ++i)
        if (cdf[i] / last > u) { idx = i; break; }
      if (idx >= n) idx = n - 1;
    }
    memcpy(centers + (int64_t)s * d, x + idx * d, sizeof(float) * d);
    kc.c = centers + (int64_t)s * d;
    kc.init = 0;
    par_rows(n, kpp_rows, &kc);
  }
  free(cdf);
  free(tmp);
  free(closest);
  return stop;
}

/* compute_tau (clustering.py:209-215): factor * mean ||f64 x - f64 c[a]|| */
double oc_tau(const float* x, int64_t n, int d, const float* c, const int32_t* labels,
              double factor) {
  double* dist = (double*)malloc(sizeof(double) * n);
  double* tmp = (double*)malloc(sizeof(double) * d);
  for (int64_t i = 0; i < n; ++i) {
    const float* cr = c + (int64_t)labels[i] * d;
    for (int t = 0; t < d; ++t) {
      const double df = (double)x[i * d + t] - (double)cr[t];
      tmp[t] = df * df;
    }
    dist[i] = sqrt(pw_d(tmp, d));
  }
  const double r = factor * (pw_d(dist, n) / (double)n);
  free(tmp);
  free(dist);
  return r;
}

/* pipeline.py:319-323: mean_i sum_t (f64 x - f64 c[a])^2 */
double oc_mse_f64(const float* x, int64_t n, int d, const float* c, const int32_t* labels) {
  double* rows = (double*)malloc(sizeof(double) * n);
  double* tmp = (double*)malloc(sizeof(double) * d);
  for (int64_t i = 0; i < n; ++i) {
    const float* cr = c + (int64_t)labels[i] * d;
    for (int t = 0; t < d; ++t) {
      const double df = (double)x[i * d + t] - (double)cr[t];
      tmp[t] = df * df;
    }
    rows[i] = pw_d(tmp, d);
  }
  const double r = pw_d(rows, n) / (double)n;
  free(tmp);
  free(rows);
  return r;
}

/* retire distances (clustering.py:292-294): f32 ||x - c[a]|| */
void oc_retire_dists(const float* x, int64_t n, int d, const float* c, const int32_t* labels,
                     float* out) {
  float* tmp = (float*)malloc(sizeof(float) * d);
  for (int64_t i = 0; i < n; ++i) {
    const float* cr = c + (int64_t)labels[i] * d;
    for (int t = 0; t < d; ++t) {
      const float df = x[i * d + t] - cr[t];
      tmp[t] = df * df;
    }
    out[i] = sqrtf(pw_f_s(tmp, d, 1));
  }
  free(tmp);
}

/* nearest_center_mse (clustering.py:203-206) */
float oc_nearest_center_mse(const float* x, int64_t n, int d, const float* c, int k) {
  int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * n);
  float* best = (float*)malloc(sizeof(float) * n);
  oc_assign(x, n, d, c, k, -1, lab, best, NULL);
  const float r = mean_f32(best, n);
  free(best);
  free(lab);
  return r;
}

/* f32 mean of an array (float(a.mean())) */
float oc_mean_f32(const float* a, int64_t n) { return mean_f32(a, n); }

/* quest.py:61-71 envelopes over member order */
void oc_envelopes(const float* x, int64_t n, int d, const int32_t* labels, int k, float* emax,
                  float* emin) {
  int64_t* seen = (int64_t*)calloc(k > 0 ? k : 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    const int j = labels[i];
    float* a = emax + (int64_t)j * d;
    float* b = emin + (int64_t)j * d;
    if (seen[j]++ == 0) {
      memcpy(a, x + i * d, sizeof(float) * d);
      memcpy(b, x + i * d, sizeof(float) * d);
    } else {
      for (int t = 0; t < d; ++t) {
        a[t] = np_max(a[t], x[i * d + t]);
        b[t] = np_min(b[t], x[i * d + t]);
      }
    }
  }
  free(seen);
}

/* quest.py:94-125 scorers: 0 quest, 1 mean, 2 clamped.  out [gq, c] */
void oc_scores(const float* reps, int gq, int d, const float* emax, const float* emin, int c,
               int scorer, float* out) {
  const int order = oc_gemm_order(gq, c, d);
  float* qa = (float*)malloc(sizeof(float) * d);
  float* qb = (float*)malloc(sizeof(float) * d);
  float* ca = (float*)malloc(sizeof(float) * d);
  float* cb = (float*)malloc(sizeof(float) * d);
  for (int g = 0; g < gq; ++g) {
    const float* q = reps + (int64_t)g * d;
    for (int t = 0; t < d; ++t) { qa[t] = np_max(q[t], 0.f); qb[t] = np_min(q[t], 0.f); }
    for (int j = 0; j < c; ++j) {
      const int hv = (g >= gq - gq % 4) && (j >= c - c % 4);
      const float* ma = emax + (int64_t)j * d;
      const float* mi = emin + (int64_t)j * d;
      float s;
      if (scorer == 1) {
        s = dot_ord(q, ma, d, order, hv);
      } else if (scorer == 2) {
        for (int t = 0; t < d; ++t) { ca[t] = np_max(ma[t], 0.f); cb[t] = np_min(ma[t], 0.f); }
        s = dot_ord(qa, ca, d, order, hv) + dot_ord(qb, cb, d, order, hv);
      } else {
        s = dot_ord(qa, ma, d, order, hv) + dot_ord(qb, mi, d, order, hv);
      }
      out[(int64_t)g * c + j] = s;
    }
  }
  free(cb);
  free(ca);
  free(qb);
  free(qa);
}

