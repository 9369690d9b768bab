/*
 * CPU ORACLE -- TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's many-RHS dichotomy path, used as the
 * CPU baseline leg of bench.py (`cpu_baseline`, `--impl reference`) and as a
 * second checker.  Never linked or called by the product path.
 *
 * Follows, function by function:
 *   lu_inplace          ref pkg/src/blocktri/_kernels.pyx:35-63  (RCOND 1e-13, first-max pivot)
 *   lu_solve_inplace    ref _kernels.pyx:66-94
 *   matmul_acc          ref _kernels.pyx:97-108
 *   thomas_factor       ref _kernels.pyx:133-170
 *   thomas_solve        ref _kernels.pyx:173-194
 *   oracle_plan_build   ref dichotomy.py:318-338 (+ 172-193 superposition, 212-236
 *                       reduced system, 28-57 tree, 134-146 / 298-304 inverse rows,
 *                       307-315 identity padding)
 *   oracle_plan_solve   ref dichotomy.py:358-390 (+ 196-209, 239-295, 345-355)
 * The reference's Cython kernels are single-threaded; this port runs its
 * independent ranges and right-hand-side columns on all
 * host threads (pthreads), reported as `cores` by bench.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

/* minimal parallel-for over independent tasks (no OpenMP runtime in this image) */
typedef void (*task_fn)(void* ctx, int64_t i);
typedef struct {
  task_fn fn;
  void* ctx;
  int64_t n;
  atomic_llong next;
} par_job;

static void* par_worker(void* arg) {
  par_job* j = (par_job*)arg;
  for (;;) {
    const int64_t i = atomic_fetch_add(&j->next, 1);
    if (i >= j->n) break;
    j->fn(j->ctx, i);
  }
  return NULL;
}

static int g_threads = 0;

int oracle_threads(void) {
  if (g_threads <= 0) {
    const char* e = getenv("ORACLE_THREADS");
    g_threads = e ? atoi(e) : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (g_threads < 1) g_threads = 1;
  }
  return g_threads;
}

static void par_for(int64_t n, task_fn fn, void* ctx) {
  int nt = oracle_threads();
  if (nt > n) nt = (int)n;
  par_job j;
  j.fn = fn;
  j.ctx = ctx;
  j.n = n;
  atomic_init(&j.next, 0);
  if (nt <= 1) {
    par_worker(&j);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
  for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, par_worker, &j);
  for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  free(th);
}

#define RCOND 1e-13

typedef struct {
  int64_t lo, hi, k;
} tnode;

typedef struct {
  int64_t n, m, P, L, npad;
  double *diag, *lower, *upper; /* padded copies: npad, npad-1, npad-1 blocks */
  double *dlu, *supper, *U, *V; /* per range: (L-1)m^2, (L-2)m^2, (L+1)m^2, (L+1)m^2 */
  int64_t* dpiv;                /* per range: (L-1)m */
  double *rd, *rl, *ru;         /* reduced system */
  int64_t nnodes;
  tnode* nodes;
  double** rows; /* inverse rows per node: m x size*m */
} oplan;

static int lu_inplace(double* a, int64_t m, int64_t* piv) {
  double tol = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += fabs(a[i * m + j]);
    if (s > tol) tol = s;
  }
  tol *= RCOND;
  for (int64_t k = 0; k < m; ++k) {
    int64_t p = k;
    double best = fabs(a[k * m + k]);
    for (int64_t i = k + 1; i < m; ++i) {
      double v = fabs(a[i * m + k]);
      if (v > best) { best = v; p = i; }
    }
    if (best <= tol) return (int)k;
    piv[k] = p;
    if (p != k)
      for (int64_t j = 0; j < m; ++j) { double t = a[k * m + j]; a[k * m + j] = a[p * m + j]; a[p * m + j] = t; }
    for (int64_t i = k + 1; i < m; ++i) {
      a[i * m + k] /= a[k * m + k];
      const double l = a[i * m + k];
      for (int64_t j = k + 1; j < m; ++j) a[i * m + j] -= l * a[k * m + j];
    }
  }
  return -1;
}

/* x: m rows of `nc` columns with row stride ldx */
static void lu_solve_inplace(const double* lu, const int64_t* piv, double* x, int64_t m, int64_t nc, int64_t ldx) {
  for (int64_t k = 0; k < m; ++k) {
    const int64_t p = piv[k];
    if (p != k)
      for (int64_t c = 0; c < nc; ++c) { double t = x[k * ldx + c]; x[k * ldx + c] = x[p * ldx + c]; x[p * ldx + c] = t; }
  }
  for (int64_t k = 1; k < m; ++k)
    for (int64_t i = 0; i < k; ++i) {
      const double v = lu[k * m + i];
      if (v != 0.0)
        for (int64_t c = 0; c < nc; ++c) x[k * ldx + c] -= v * x[i * ldx + c];
    }
  for (int64_t k = m - 1; k >= 0; --k) {
    for (int64_t i = k + 1; i < m; ++i) {
      const double v = lu[k * m + i];
      if (v != 0.0)
        for (int64_t c = 0; c < nc; ++c) x[k * ldx + c] -= v * x[i * ldx + c];
    }
    const double d = lu[k * m + k];
    for (int64_t c = 0; c < nc; ++c) x[k * ldx + c] /= d;
  }
}

/* out (m x nc, ld lo) += sign * a (m x kk, ld kk) @ b (kk x nc, ld lb) */
static void matmul_acc(const double* a, const double* b, double* out, int64_t m, int64_t kk, int64_t nc,
                       int64_t lb, int64_t lo, double sign) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = 0; k < kk; ++k) {
      const double v = sign * a[i * kk + k];
      if (v == 0.0) continue;
      const double* br = b + k * lb;
      double* orow = out + i * lo;
      for (int64_t c = 0; c < nc; ++c) orow[c] += v * br[c];
    }
}

/* returns failing local row or -1 */
static int64_t thomas_factor(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m,
                             double* dlu, int64_t* dpiv, double* supper) {
  const int64_t b = m * m;
  memcpy(dlu, diag, sizeof(double) * b);
  for (int64_t i = 0; i < n; ++i) {
    if (lu_inplace(dlu + i * b, m, dpiv + i * m) >= 0) return i;
    if (i < n - 1) {
      memcpy(supper + i * b, upper + i * b, sizeof(double) * b);
      lu_solve_inplace(dlu + i * b, dpiv + i * m, supper + i * b, m, m, m);
      memcpy(dlu + (i + 1) * b, diag + (i + 1) * b, sizeof(double) * b);
      matmul_acc(lower + i * b, supper + i * b, dlu + (i + 1) * b, m, m, m, m, m, -1.0);
    }
  }
  return -1;
}

/* x: n blocks of m rows x nc columns, block stride m*ldx, row stride ldx (in place) */
static void thomas_solve(const double* dlu, const int64_t* dpiv, const double* supper, const double* lower, int64_t n,
                         int64_t m, double* x, int64_t nc, int64_t ldx) {
  const int64_t b = m * m, xb = m * ldx;
  lu_solve_inplace(dlu, dpiv, x, m, nc, ldx);
  for (int64_t i = 1; i < n; ++i) {
    matmul_acc(lower + (i - 1) * b, x + (i - 1) * xb, x + i * xb, m, m, nc, ldx, ldx, 1.0);
    lu_solve_inplace(dlu + i * b, dpiv + i * m, x + i * xb, m, nc, ldx);
  }
  for (int64_t i = n - 2; i >= 0; --i) matmul_acc(supper + i * b, x + (i + 1) * xb, x + i * xb, m, m, nc, ldx, ldx, 1.0);
}

static void transpose_blocks(const double* src, double* dst, int64_t cnt, int64_t m) {
  for (int64_t q = 0; q < cnt; ++q)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < m; ++j) dst[q * m * m + j * m + i] = src[q * m * m + i * m + j];
}

void oracle_plan_free(oplan* p) {
  if (!p) return;
  free(p->diag); free(p->lower); free(p->upper); free(p->dlu); free(p->supper); free(p->U); free(p->V);
  free(p->dpiv); free(p->rd); free(p->rl); free(p->ru);
  if (p->rows)
    for (int64_t i = 0; i < p->nnodes; ++i) free(p->rows[i]);
  free(p->rows); free(p->nodes);
  free(p);
}


typedef struct {
  oplan* p;
  int64_t* fail;
} build_ctx;

/* superposition factors of one range (ref dichotomy.py:172-193) */
static void build_range(void* vctx, int64_t q) {
  build_ctx* c = (build_ctx*)vctx;
  oplan* p = c->p;
  const int64_t m = p->m, b = m * m, L = p->L, npad = p->npad, lo = q * L, hi = lo + L;
  const int64_t ni = L >= 2 ? L - 1 : 0;
  double* U = p->U + q * (L + 1) * b;
  double* V = p->V + q * (L + 1) * b;
  c->fail[q] = -1;
  for (int64_t d = 0; d < m; ++d) { U[d * m + d] = 1.0; V[L * b + d * m + d] = 1.0; }
  if (L < 2) return;
  double* dlu = p->dlu + q * ni * b;
  int64_t* dpiv = p->dpiv + q * ni * m;
  double* sup = p->supper + q * (ni > 1 ? ni - 1 : 1) * b;
  const int64_t f = thomas_factor(p->diag + (lo + 1) * b, p->lower + (lo + 1) * b, p->upper + (lo + 1) * b, ni, m,
                                  dlu, dpiv, sup);
  if (f >= 0) { c->fail[q] = f; return; }
  memcpy(U + b, p->lower + lo * b, sizeof(double) * b); /* rhs e0 (x) A_{lo+1} */
  thomas_solve(dlu, dpiv, sup, p->lower + (lo + 1) * b, ni, m, U + b, m, m);
  if (hi - 1 < npad - 1) memcpy(V + (L - 1) * b, p->upper + (hi - 1) * b, sizeof(double) * b);
  thomas_solve(dlu, dpiv, sup, p->lower + (lo + 1) * b, ni, m, V + b, m, m);
}

typedef struct {
  const oplan* p;
  const double* fp;
  double* W;
  double* xp;
  const double* xt;
  int64_t k, cch, nch;
} solve_ctx;

/* particular solution W of one (range, column chunk) (ref dichotomy.py:196-209) */
static void solve_w(void* vctx, int64_t task) {
  solve_ctx* c = (solve_ctx*)vctx;
  const oplan* p = c->p;
  const int64_t m = p->m, b = m * m, L = p->L, k = c->k, mk = m * k, ni = L >= 2 ? L - 1 : 0;
  const int64_t q = task / c->nch, ch = task % c->nch;
  if (L < 2) return;
  const int64_t c0 = ch * c->cch, nc = (c0 + c->cch <= k) ? c->cch : k - c0;
  double* w = c->W + q * (L + 1) * mk + mk + c0;
  for (int64_t r = 0; r < ni; ++r)
    for (int64_t i = 0; i < m; ++i) memcpy(w + r * mk + i * k, c->fp + (q * L + 1 + r) * mk + i * k + c0, sizeof(double) * nc);
  thomas_solve(p->dlu + q * ni * b, p->dpiv + q * ni * m, p->supper + q * (ni > 1 ? ni - 1 : 1) * b,
               p->lower + (q * L + 1) * b, ni, m, w, nc, k);
}

/* recovery of one range: x = U x~_q + V x~_{q+1} + W (ref dichotomy.py:345-355) */
static void solve_recover(void* vctx, int64_t q) {
  solve_ctx* c = (solve_ctx*)vctx;
  const oplan* p = c->p;
  const int64_t m = p->m, b = m * m, L = p->L, k = c->k, mk = m * k, K = q * L;
  memcpy(c->xp + K * mk, c->xt + q * mk, sizeof(double) * mk);
  for (int64_t r = 1; r < L; ++r) {
    double* o = c->xp + (K + r) * mk;
    memcpy(o, c->W + q * (L + 1) * mk + r * mk, sizeof(double) * mk);
    matmul_acc(p->U + q * (L + 1) * b + r * b, c->xt + q * mk, o, m, m, k, k, k, 1.0);
    matmul_acc(p->V + q * (L + 1) * b + r * b, c->xt + (q + 1) * mk, o, m, m, k, k, k, 1.0);
  }
}

/* status: 0 ok, 2 singular pivot (*err_row = local row), 3 invalid ranks */
int oracle_plan_build(const double* diag, const double* lower, const double* upper, int64_t n, int64_t m, int64_t P,
                      oplan** out, int64_t* err_row) {
  *out = NULL;
  *err_row = -1;
  if (P < 1 || P > n) return 3;
  oplan* p = (oplan*)calloc(1, sizeof(oplan));
  const int64_t b = m * m, L = (n + P - 1) / P, npad = L * P;
  p->n = n; p->m = m; p->P = P; p->L = L; p->npad = npad;
  p->diag = (double*)calloc((size_t)npad * b, sizeof(double));
  p->lower = (double*)calloc((size_t)(npad > 1 ? npad - 1 : 1) * b, sizeof(double));
  p->upper = (double*)calloc((size_t)(npad > 1 ? npad - 1 : 1) * b, sizeof(double));
  memcpy(p->diag, diag, sizeof(double) * n * b);
  for (int64_t i = n; i < npad; ++i)
    for (int64_t d = 0; d < m; ++d) p->diag[i * b + d * m + d] = 1.0;
  if (n > 1) {
    memcpy(p->lower, lower, sizeof(double) * (n - 1) * b);
    memcpy(p->upper, upper, sizeof(double) * (n - 1) * b);
  }
  const int64_t ni = L >= 2 ? L - 1 : 0;
  p->dlu = (double*)calloc((size_t)P * (ni ? ni : 1) * b, sizeof(double));
  p->dpiv = (int64_t*)calloc((size_t)P * (ni ? ni : 1) * m, sizeof(int64_t));
  p->supper = (double*)calloc((size_t)P * (ni > 1 ? ni - 1 : 1) * b, sizeof(double));
  p->U = (double*)calloc((size_t)P * (L + 1) * b, sizeof(double));
  p->V = (double*)calloc((size_t)P * (L + 1) * b, sizeof(double));
  int64_t* fail = (int64_t*)malloc(sizeof(int64_t) * P);
  build_ctx bc = {p, fail};
  par_for(P, build_range, &bc);
  for (int64_t q = 0; q < P; ++q)
    if (fail[q] >= 0) { *err_row = fail[q]; free(fail); oracle_plan_free(p); return 2; }
  free(fail);
  /* reduced system (ref dichotomy.py:212-236) */
  p->rd = (double*)calloc((size_t)P * b, sizeof(double));
  p->rl = (double*)calloc((size_t)(P > 1 ? P - 1 : 1) * b, sizeof(double));
  p->ru = (double*)calloc((size_t)(P > 1 ? P - 1 : 1) * b, sizeof(double));
  for (int64_t q = 0; q < P; ++q) {
    const int64_t K = q * L;
    double* d = p->rd + q * b;
    memcpy(d, p->diag + K * b, sizeof(double) * b);
    if (q >= 1) {
      const double* Vp = p->V + (q - 1) * (L + 1) * b + (L - 1) * b;
      const double* Up = p->U + (q - 1) * (L + 1) * b + (L - 1) * b;
      matmul_acc(p->lower + (K - 1) * b, Vp, d, m, m, m, m, m, -1.0);
      matmul_acc(p->lower + (K - 1) * b, Up, p->rl + (q - 1) * b, m, m, m, m, m, 1.0);
    }
    if (K < npad - 1) {
      matmul_acc(p->upper + K * b, p->U + q * (L + 1) * b + b, d, m, m, m, m, m, -1.0);
      if (q <= P - 2) matmul_acc(p->upper + K * b, p->V + q * (L + 1) * b + b, p->ru + q * b, m, m, m, m, m, 1.0);
    }
  }
  /* partition tree, BFS, split k = lo + (hi-lo+1)/2 (ref dichotomy.py:28-57) */
  p->nodes = (tnode*)malloc(sizeof(tnode) * P);
  int64_t head = 0, tail = 0;
  p->nodes[tail++] = (tnode){0, P - 1, 0};
  while (head < tail) {
    tnode* t = &p->nodes[head++];
    t->k = t->lo + (t->hi - t->lo + 1) / 2;
    if (t->k - 1 >= t->lo) p->nodes[tail++] = (tnode){t->lo, t->k - 1, 0};
    if (t->k + 1 <= t->hi) p->nodes[tail++] = (tnode){t->k + 1, t->hi, 0};
  }
  p->nnodes = tail;
  p->rows = (double**)calloc(p->nnodes, sizeof(double*));
  /* inverse rows by transposed sweeps with unit RHS (ref dichotomy.py:134-146) */
  int64_t tfail_node = -1, tfail_row = -1;
  for (int64_t t = 0; t < p->nnodes; ++t) {
    const int64_t lo = p->nodes[t].lo, hi = p->nodes[t].hi, s = hi - lo + 1, kk = p->nodes[t].k - lo;
    double* sd = (double*)malloc(sizeof(double) * s * b);
    double* sl = (double*)malloc(sizeof(double) * (s > 1 ? s - 1 : 1) * b);
    double* su = (double*)malloc(sizeof(double) * (s > 1 ? s - 1 : 1) * b);
    transpose_blocks(p->rd + lo * b, sd, s, m);
    if (s > 1) {
      transpose_blocks(p->ru + lo * b, sl, s - 1, m); /* transpose swaps couplings (ref core.py:137-143) */
      transpose_blocks(p->rl + lo * b, su, s - 1, m);
    }
    double* tdlu = (double*)malloc(sizeof(double) * s * b);
    int64_t* tpiv = (int64_t*)malloc(sizeof(int64_t) * s * m);
    double* tsup = (double*)malloc(sizeof(double) * (s > 1 ? s - 1 : 1) * b);
    const int64_t f = thomas_factor(sd, sl, su, s, m, tdlu, tpiv, tsup);
    if (f >= 0) {
      tfail_node = t; tfail_row = f;
      free(sd); free(sl); free(su); free(tdlu); free(tpiv); free(tsup);
      break;
    }
    double* y = (double*)calloc((size_t)s * b, sizeof(double));
    for (int64_t d = 0; d < m; ++d) y[kk * b + d * m + d] = 1.0;
    thomas_solve(tdlu, tpiv, tsup, sl, s, m, y, m, m);
    double* R = (double*)malloc(sizeof(double) * s * b);
    for (int64_t a = 0; a < m; ++a)
      for (int64_t i = 0; i < s; ++i)
        for (int64_t c = 0; c < m; ++c) R[a * s * m + i * m + c] = y[i * b + c * m + a];
    p->rows[t] = R;
    free(y); free(sd); free(sl); free(su); free(tdlu); free(tpiv); free(tsup);
  }
  if (tfail_node >= 0) { *err_row = tfail_row; oracle_plan_free(p); return 2; }
  *out = p;
  return 0;
}

/* f, x: (n, m, k) row-major; x may not alias f */
int oracle_plan_solve(const oplan* p, const double* f, double* x, int64_t k) {
  const int64_t n = p->n, m = p->m, P = p->P, L = p->L, npad = p->npad, b = m * m, mk = m * k;
  double* fp = (double*)calloc((size_t)npad * mk, sizeof(double));
  memcpy(fp, f, sizeof(double) * n * mk);
  double* W = (double*)calloc((size_t)P * (L + 1) * mk, sizeof(double));
  /* particular solutions W per range and column chunk (ref dichotomy.py:196-209) */
  const int64_t cch = k >= 64 ? 16 : (k >= 8 ? 4 : 1);
  solve_ctx sc = {p, fp, W, NULL, NULL, k, cch, (k + cch - 1) / cch};
  par_for(P * sc.nch, solve_w, &sc);
  /* interface RHS (ref dichotomy.py:239-276) */
  double* ft = (double*)calloc((size_t)P * mk, sizeof(double));
  for (int64_t q = 0; q < P; ++q) {
    const int64_t K = q * L;
    memcpy(ft + q * mk, fp + K * mk, sizeof(double) * mk);
    if (K < npad - 1) matmul_acc(p->upper + K * b, W + q * (L + 1) * mk + mk, ft + q * mk, m, m, k, k, k, 1.0);
    if (q >= 1) matmul_acc(p->lower + (K - 1) * b, W + (q - 1) * (L + 1) * mk + (L - 1) * mk, ft + q * mk, m, m, k, k, k, 1.0);
  }
  /* Algorithm 1 (ref dichotomy.py:279-295) */
  double* xt = (double*)calloc((size_t)(P + 1) * mk, sizeof(double));
  for (int64_t t = 0; t < p->nnodes; ++t) {
    const int64_t lo = p->nodes[t].lo, hi = p->nodes[t].hi, kk = p->nodes[t].k, s = hi - lo + 1;
    double* xk = xt + kk * mk;
    memset(xk, 0, sizeof(double) * mk);
    matmul_acc(p->rows[t], ft + lo * mk, xk, m, s * m, k, k, k, 1.0);
    if (kk - 1 >= lo) matmul_acc(p->ru + (kk - 1) * b, xk, ft + (kk - 1) * mk, m, m, k, k, k, 1.0);
    if (kk + 1 <= hi) matmul_acc(p->rl + kk * b, xk, ft + (kk + 1) * mk, m, m, k, k, k, 1.0);
  }
  /* recovery x = U x~_q + V x~_{q+1} + W (ref dichotomy.py:345-355) */
  double* xp = (double*)calloc((size_t)npad * mk, sizeof(double));
  sc.xp = xp;
  sc.xt = xt;
  par_for(P, solve_recover, &sc);
  memcpy(x, xp, sizeof(double) * n * mk);
  free(fp); free(W); free(ft); free(xt); free(xp);
  return 0;
}
