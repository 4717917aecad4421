/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 streaming path.
 *
 * A plain-C restatement of the reference's per-slice streaming ST-HOSVD path
 * (arXiv 2308.16395, Alg. 2), written against the reference proj/src sources.
 * Every function cites the reference lines it follows. Floating-point
 * operations are issued in the same order as the reference so that, built
 * with the same flags (-O3, no FMA contraction), results are bit-identical
 * to the reference itself; tests/test_oracle.py pins that against
 * oracle/_ref (the reference compiled in place) and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product (paper_2308_16395_b200/libtsg.so) never
 * links or calls it.
 *
 * Layouts (reference tensor.hpp:11-19, matrix.hpp:15-50):
 *   tensors colexicographic (mode 0 fastest); matrices column-major;
 *   the streaming factor ("left") row-major n_d x r (isvd.hpp:18-60);
 *   right (Q) column-major n x r and bit-identical to v_tensor's buffer
 *   (streaming.cpp:19-35).
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC(name) tko_##name
#include "oracle_abi.h"

#define MAXD ORC_MAXD

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];
static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
const char* tko_last_error(void) { return g_err; }

enum { OK = 0, EINVAL_ = 1, EDRIFT = 2, EOTHER = 3 };

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}

/* ------------------------------------------------------------- containers */
typedef struct { size_t rows, cols; double* a; } mat; /* column-major */
typedef struct { int order; size_t dims[MAXD]; size_t size; double* a; } ten;

static mat mat_new(size_t r, size_t c) {
  mat m = {r, c, (double*)xcalloc(r * c, sizeof(double))};
  return m;
}
static void mat_free(mat* m) { free(m->a); m->a = NULL; m->rows = m->cols = 0; }
#define M(m, i, j) ((m).a[(size_t)(j) * (m).rows + (i)])

static ten ten_new(int order, const size_t* dims) {
  ten t;
  t.order = order;
  t.size = 1;
  for (int k = 0; k < order; ++k) { t.dims[k] = dims[k]; t.size *= dims[k]; }
  t.a = (double*)xcalloc(t.size, sizeof(double));
  return t;
}
static void ten_free(ten* t) { free(t->a); t->a = NULL; t->size = 0; }
static ten ten_copy(const ten* s) {
  ten t = ten_new(s->order, s->dims);
  memcpy(t.a, s->a, s->size * sizeof(double));
  return t;
}

/* Pairwise sum of squares, leaf 64 (matrix.cpp:14-22). */
static double sumsq(const double* p, size_t n) {
  if (n <= 64) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += p[i] * p[i];
    return s;
  }
  size_t half = n / 2;
  return sumsq(p, half) + sumsq(p + half, n - half);
}
double tko_sum_of_squares(const double* p, int64_t n) { return sumsq(p, (size_t)n); }

static double ten_norm(const ten* t) { return sqrt(sumsq(t->a, t->size)); }

/* Block shape around a mode (tensor.cpp:26-34). */
static void blocks_around(const ten* t, int mode, size_t* left, size_t* right) {
  *left = 1; *right = 1;
  for (int l = 0; l < mode; ++l) *left *= t->dims[l];
  for (int l = mode + 1; l < t->order; ++l) *right *= t->dims[l];
}

/* multiply(a, b, ta, tb) (matrix.cpp:32-86). */
static mat multiply(const mat* a, const mat* b, int ta, int tb) {
  size_t m = ta ? a->cols : a->rows, k = ta ? a->rows : a->cols;
  size_t n = tb ? b->rows : b->cols;
  mat c = mat_new(m, n);
  if (m == 0 || n == 0 || k == 0) return c;
  if (!ta && !tb) {
    for (size_t j = 0; j < n; ++j) {
      double* cj = c.a + j * m;
      for (size_t l = 0; l < k; ++l) {
        double blj = M(*b, l, j);
        if (blj == 0.0) continue;
        const double* al = a->a + l * a->rows;
        for (size_t i = 0; i < m; ++i) cj[i] += al[i] * blj;
      }
    }
  } else if (ta && !tb) {
    for (size_t j = 0; j < n; ++j) {
      const double* bj = b->a + j * b->rows;
      double* cj = c.a + j * m;
      for (size_t i = 0; i < m; ++i) {
        const double* ai = a->a + i * a->rows;
        double s = 0.0;
        for (size_t l = 0; l < k; ++l) s += ai[l] * bj[l];
        cj[i] = s;
      }
    }
  } else if (!ta && tb) {
    for (size_t l = 0; l < k; ++l) {
      const double* al = a->a + l * a->rows;
      for (size_t j = 0; j < n; ++j) {
        double bjl = M(*b, j, l);
        if (bjl == 0.0) continue;
        double* cj = c.a + j * m;
        for (size_t i = 0; i < m; ++i) cj[i] += al[i] * bjl;
      }
    }
  } else {
    for (size_t j = 0; j < n; ++j) {
      double* cj = c.a + j * m;
      for (size_t i = 0; i < m; ++i) {
        const double* ai = a->a + i * a->rows;
        double s = 0.0;
        for (size_t l = 0; l < k; ++l) s += ai[l] * M(*b, j, l);
        cj[i] = s;
      }
    }
  }
  return c;
}

/* hcat (matrix.cpp:97-112). */
static mat hcat(const mat* a, const mat* b) {
  if (a->rows * a->cols == 0 && a->rows == 0) {
    mat c = mat_new(b->rows, b->cols);
    memcpy(c.a, b->a, b->rows * b->cols * sizeof(double));
    return c;
  }
  if (b->rows * b->cols == 0 && b->rows == 0) {
    mat c = mat_new(a->rows, a->cols);
    memcpy(c.a, a->a, a->rows * a->cols * sizeof(double));
    return c;
  }
  mat c = mat_new(a->rows, a->cols + b->cols);
  memcpy(c.a, a->a, a->rows * a->cols * sizeof(double));
  memcpy(c.a + a->rows * a->cols, b->a, b->rows * b->cols * sizeof(double));
  return c;
}

/* orthonormality_defect (matrix.cpp:118-131). */
static double orth_defect(const mat* m) {
  double worst = 0.0;
  for (size_t j = 0; j < m->cols; ++j) {
    const double* cj = m->a + j * m->rows;
    for (size_t i = 0; i <= j; ++i) {
      const double* ci = m->a + i * m->rows;
      double dot = 0.0;
      for (size_t l = 0; l < m->rows; ++l) dot += ci[l] * cj[l];
      double target = (i == j) ? 1.0 : 0.0;
      double d = fabs(dot - target);
      if (d > worst) worst = d;
    }
  }
  return worst;
}

/* unfold (tensor.cpp:67-84). */
static mat unfold(const ten* t, int mode) {
  size_t n = t->dims[mode];
  size_t cols = (n == 0) ? 0 : t->size / n;
  mat m = mat_new(n, cols);
  size_t left, right;
  blocks_around(t, mode, &left, &right);
  for (size_t r = 0; r < right; ++r) {
    const double* slab = t->a + r * left * n;
    for (size_t l = 0; l < left; ++l) {
      double* dst = m.a + (l + r * left) * n;
      for (size_t i = 0; i < n; ++i) dst[i] = slab[l + i * left];
    }
  }
  return m;
}

/* ttm (tensor.cpp:106-162), including the mode-0 fast path. */
static ten ttm(const ten* t, int mode, const mat* a, int transpose_a) {
  size_t n = t->dims[mode];
  size_t produced = transpose_a ? a->cols : a->rows;
  size_t od[MAXD];
  for (int k = 0; k < t->order; ++k) od[k] = t->dims[k];
  od[mode] = produced;
  ten out = ten_new(t->order, od);
  size_t left, right;
  blocks_around(t, mode, &left, &right);
  if (mode == 0) {
    for (size_t r = 0; r < right; ++r) {
      const double* x = t->a + r * n;
      double* y = out.a + r * produced;
      if (transpose_a) {
        for (size_t j = 0; j < produced; ++j) {
          const double* ajc = a->a + j * a->rows;
          double s = 0.0;
          for (size_t i = 0; i < n; ++i) s += ajc[i] * x[i];
          y[j] = s;
        }
      } else {
        for (size_t i = 0; i < n; ++i) {
          double xi = x[i];
          if (xi == 0.0) continue;
          const double* aic = a->a + i * a->rows;
          for (size_t j = 0; j < produced; ++j) y[j] += aic[j] * xi;
        }
      }
    }
    return out;
  }
  for (size_t r = 0; r < right; ++r) {
    const double* src = t->a + r * left * n;
    double* dst = out.a + r * left * produced;
    for (size_t i = 0; i < n; ++i) {
      const double* si = src + i * left;
      for (size_t j = 0; j < produced; ++j) {
        double w = transpose_a ? M(*a, i, j) : M(*a, j, i);
        if (w == 0.0) continue;
        double* dj = dst + j * left;
        for (size_t l = 0; l < left; ++l) dj[l] += si[l] * w;
      }
    }
  }
  return out;
}

/* pad_with_zeros (tensor.cpp:168-184). */
static ten pad_with_zeros(const ten* t, int mode, size_t extra) {
  size_t od[MAXD];
  for (int k = 0; k < t->order; ++k) od[k] = t->dims[k];
  od[mode] += extra;
  ten out = ten_new(t->order, od);
  size_t n = t->dims[mode], left, right;
  blocks_around(t, mode, &left, &right);
  for (size_t r = 0; r < right; ++r)
    memcpy(out.a + r * left * (n + extra), t->a + r * left * n,
           left * n * sizeof(double));
  return out;
}

/* concat_along_mode (tensor.cpp:186-209). */
static ten concat_along_mode(int mode, const ten* a, const ten* b) {
  size_t od[MAXD];
  for (int k = 0; k < a->order; ++k) od[k] = a->dims[k];
  od[mode] += b->dims[mode];
  ten out = ten_new(a->order, od);
  size_t na = a->dims[mode], nb = b->dims[mode], left, right;
  blocks_around(a, mode, &left, &right);
  for (size_t r = 0; r < right; ++r) {
    double* dst = out.a + r * left * (na + nb);
    memcpy(dst, a->a + r * left * na, left * na * sizeof(double));
    memcpy(dst + left * na, b->a + r * left * nb, left * nb * sizeof(double));
  }
  return out;
}

/* ----------------------------------------------------------------- linalg */
/* gram_from_cols (linalg.cpp:80-94): rows x rows. */
static mat gram_from_cols(const double* a, size_t rows, size_t cols) {
  mat g = mat_new(rows, rows);
  for (size_t c = 0; c < cols; ++c) {
    const double* ac = a + c * rows;
    for (size_t j = 0; j < rows; ++j) {
      double w = ac[j];
      if (w == 0.0) continue;
      double* gj = g.a + j * rows;
      for (size_t i = 0; i <= j; ++i) gj[i] += ac[i] * w;
    }
  }
  for (size_t j = 0; j < rows; ++j)
    for (size_t i = 0; i < j; ++i) M(g, j, i) = M(g, i, j);
  return g;
}

/* gram_transposed_from_cols (linalg.cpp:100-114): cols x cols. */
static mat gram_t_from_cols(const double* a, size_t rows, size_t cols) {
  mat g = mat_new(cols, cols);
  for (size_t j = 0; j < cols; ++j) {
    const double* aj = a + j * rows;
    for (size_t i = 0; i <= j; ++i) {
      const double* ai = a + i * rows;
      double dot = 0.0;
      for (size_t l = 0; l < rows; ++l) dot += ai[l] * aj[l];
      M(g, i, j) = dot;
      M(g, j, i) = dot;
    }
  }
  return g;
}

/* off_diagonal_norm (linalg.cpp:18-24). */
static double off_norm(const mat* g) {
  double s = 0.0;
  for (size_t j = 0; j < g->cols; ++j)
    for (size_t i = 0; i < g->rows; ++i)
      if (i != j) s += M(*g, i, j) * M(*g, i, j);
  return sqrt(s);
}

/* One Jacobi rotation zeroing g(p,q) (linalg.cpp:27-60). */
static void rotate(mat* g, mat* v, size_t p, size_t q) {
  double gpq = M(*g, p, q);
  if (gpq == 0.0) return;
  double theta = (M(*g, q, q) - M(*g, p, p)) / (2.0 * gpq);
  double t = (theta >= 0.0) ? 1.0 / (theta + sqrt(1.0 + theta * theta))
                            : 1.0 / (theta - sqrt(1.0 + theta * theta));
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = t * c;
  size_t n = g->rows;
  double gpp = M(*g, p, p), gqq = M(*g, q, q);
  for (size_t i = 0; i < n; ++i) {
    if (i == p || i == q) continue;
    double gip = M(*g, i, p), giq = M(*g, i, q);
    M(*g, i, p) = c * gip - s * giq;
    M(*g, p, i) = M(*g, i, p);
    M(*g, i, q) = s * gip + c * giq;
    M(*g, q, i) = M(*g, i, q);
  }
  M(*g, p, p) = gpp - t * gpq;
  M(*g, q, q) = gqq + t * gpq;
  M(*g, p, q) = 0.0;
  M(*g, q, p) = 0.0;
  for (size_t i = 0; i < v->rows; ++i) {
    double vip = M(*v, i, p), viq = M(*v, i, q);
    M(*v, i, p) = c * vip - s * viq;
    M(*v, i, q) = s * vip + c * viq;
  }
}

/* sym_eig_desc (linalg.cpp:120-181): cyclic row-order Jacobi, stable
 * descending sort, negative clamp, largest-|entry|-positive sign rule. */
static int sym_eig_desc(const mat* gin, double* evals, mat* evecs) {
  size_t n = gin->rows;
  double max_abs = 0.0, max_asym = 0.0;
  for (size_t j = 0; j < n; ++j)
    for (size_t i = 0; i < n; ++i) {
      double a = fabs(M(*gin, i, j));
      double s = fabs(M(*gin, i, j) - M(*gin, j, i));
      if (a > max_abs) max_abs = a;
      if (s > max_asym) max_asym = s;
    }
  if (max_asym > 1e-10 * (max_abs > 1e-300 ? max_abs : 1e-300)) {
    set_err("sym_eig_desc: matrix is not symmetric");
    return EINVAL_;
  }
  mat g = mat_new(n, n);
  memcpy(g.a, gin->a, n * n * sizeof(double));
  mat v = mat_new(n, n);
  for (size_t i = 0; i < n; ++i) M(v, i, i) = 1.0;
  double tol = 1e-14 * sqrt(sumsq(gin->a, n * n));
  for (int sweep = 0; sweep < 30; ++sweep) {
    if (off_norm(&g) <= tol) break;
    for (size_t p = 0; p + 1 < n; ++p)
      for (size_t q = p + 1; q < n; ++q) rotate(&g, &v, p, q);
  }
  /* stable sort by descending diagonal (std::stable_sort equivalent) */
  size_t* order = (size_t*)xcalloc(n, sizeof(size_t));
  for (size_t i = 0; i < n; ++i) order[i] = i;
  for (size_t i = 1; i < n; ++i) {
    size_t key = order[i];
    double kv = M(g, key, key);
    size_t j = i;
    while (j > 0 && kv > M(g, order[j - 1], order[j - 1])) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = key;
  }
  double scale = 0.0;
  for (size_t j = 0; j < n; ++j) {
    double a = fabs(M(g, order[j], order[j]));
    if (a > scale) scale = a;
  }
  *evecs = mat_new(n, n);
  for (size_t j = 0; j < n; ++j) {
    double lambda = M(g, order[j], order[j]);
    if (lambda < 0.0) lambda = 0.0; /* warn below -1e-12*scale (log only) */
    evals[j] = lambda;
    const double* src = v.a + order[j] * n;
    double* dst = evecs->a + j * n;
    memcpy(dst, src, n * sizeof(double));
    size_t arg = 0;
    for (size_t i = 1; i < n; ++i)
      if (fabs(dst[i]) > fabs(dst[arg])) arg = i;
    if (n > 0 && dst[arg] < 0.0)
      for (size_t i = 0; i < n; ++i) dst[i] = -dst[i];
  }
  (void)scale;
  free(order);
  mat_free(&g);
  mat_free(&v);
  return OK;
}

/* truncation_rank (linalg.cpp:183-208). Returns (size_t)-1 on error. */
static size_t truncation_rank(const double* ev, size_t n, double delta) {
  if (delta < 0.0) { set_err("truncation_rank: delta must be nonnegative"); return (size_t)-1; }
  for (size_t i = 0; i < n; ++i) {
    if (ev[i] < 0.0) { set_err("truncation_rank: eigenvalues must be nonnegative"); return (size_t)-1; }
    if (i > 0 && ev[i] > ev[i - 1]) { set_err("truncation_rank: eigenvalues must be descending"); return (size_t)-1; }
  }
  if (n == 0) return 0;
  double* trailing = (double*)xcalloc(n + 1, sizeof(double));
  for (size_t i = n; i-- > 0;) trailing[i] = trailing[i + 1] + ev[i];
  double budget = delta * delta;
  size_t res = n;
  for (size_t r = 0; r <= n; ++r)
    if (trailing[r] <= budget) { res = r < 1 ? 1 : r; break; }
  free(trailing);
  return res;
}

/* orthonormalize_columns: one MGS pass (linalg.cpp:64-78). */
static void orthonormalize_columns(mat* u) {
  size_t n = u->rows;
  for (size_t j = 0; j < u->cols; ++j) {
    double* uj = u->a + j * n;
    for (size_t i = 0; i < j; ++i) {
      const double* ui = u->a + i * n;
      double dot = 0.0;
      for (size_t l = 0; l < n; ++l) dot += ui[l] * uj[l];
      for (size_t l = 0; l < n; ++l) uj[l] -= dot * ui[l];
    }
    double norm = sqrt(sumsq(uj, n));
    if (norm > 0.0)
      for (size_t l = 0; l < n; ++l) uj[l] /= norm;
  }
}

typedef struct { mat left, right; double* sigma; size_t rank; double discarded; } smallsvd;

/* small_svd_truncated (linalg.cpp:210-259): Gram route. */
static int small_svd_truncated(const mat* m, double thr, smallsvd* out) {
  memset(out, 0, sizeof *out);
  if (thr < 0.0) { set_err("small_svd_truncated: threshold must be nonnegative"); return EINVAL_; }
  if (m->rows == 0 || m->cols == 0) {
    out->left = mat_new(m->rows, 0);
    out->right = mat_new(m->cols, 0);
    out->sigma = (double*)xcalloc(1, sizeof(double));
    return OK;
  }
  mat g = gram_t_from_cols(m->a, m->rows, m->cols);
  size_t n = m->cols;
  double* lambda = (double*)xcalloc(n, sizeof(double));
  mat vecs;
  int st = sym_eig_desc(&g, lambda, &vecs);
  mat_free(&g);
  if (st) { free(lambda); return st; }
  double smax = sqrt(lambda[0]);
  if (smax == 0.0) {
    out->left = mat_new(m->rows, 0);
    out->right = mat_new(m->cols, 0);
    out->sigma = (double*)xcalloc(1, sizeof(double));
    free(lambda);
    mat_free(&vecs);
    return OK;
  }
  double floor_ = 1e-14 * smax;
  for (size_t i = 0; i < n; ++i)
    if (sqrt(lambda[i]) <= floor_) lambda[i] = 0.0;
  size_t rank = truncation_rank(lambda, n, thr);
  if (rank == (size_t)-1) { free(lambda); mat_free(&vecs); return EINVAL_; }
  out->discarded = 0.0;
  for (size_t j = n; j-- > rank;) out->discarded += lambda[j];
  out->rank = rank;
  out->sigma = (double*)xcalloc(rank, sizeof(double));
  out->right = mat_new(n, rank);
  for (size_t j = 0; j < rank; ++j) {
    out->sigma[j] = sqrt(lambda[j]);
    memcpy(out->right.a + j * n, vecs.a + j * n, n * sizeof(double));
  }
  out->left = multiply(m, &out->right, 0, 0);
  for (size_t j = 0; j < rank; ++j) {
    double* uj = out->left.a + j * m->rows;
    double inv = 1.0 / out->sigma[j];
    for (size_t i = 0; i < m->rows; ++i) uj[i] *= inv;
  }
  orthonormalize_columns(&out->left);
  free(lambda);
  mat_free(&vecs);
  return OK;
}

static void smallsvd_free(smallsvd* s) {
  mat_free(&s->left);
  mat_free(&s->right);
  free(s->sigma);
  s->sigma = NULL;
}

/* trailing_sum (sthosvd.cpp:31-35). */
static double trailing_sum(const double* v, size_t n, size_t from) {
  double s = 0.0;
  for (size_t i = n; i-- > from;) s += v[i];
  return s;
}

typedef struct { mat basis; double* evals; size_t n_evals; double discarded; } subspace;

/* mode_subspace (sthosvd.cpp:39-92): Gram route when rows <= cols, else the
 * thin route through the transposed Gram with back-substitution + MGS. */
static int mode_subspace(const ten* t, int mode, double delta, subspace* out) {
  memset(out, 0, sizeof *out);
  size_t rows = t->dims[mode];
  size_t cols = rows == 0 ? 0 : t->size / rows;
  if (rows <= cols) {
    mat g;
    if (mode == 0) {
      g = gram_from_cols(t->a, rows, cols);
    } else {
      mat u = unfold(t, mode);
      g = gram_from_cols(u.a, u.rows, u.cols);
      mat_free(&u);
    }
    out->evals = (double*)xcalloc(rows, sizeof(double));
    out->n_evals = rows;
    mat vecs;
    int st = sym_eig_desc(&g, out->evals, &vecs);
    mat_free(&g);
    if (st) return st;
    size_t rank = truncation_rank(out->evals, rows, delta);
    if (rank == (size_t)-1) { mat_free(&vecs); return EINVAL_; }
    out->discarded = trailing_sum(out->evals, rows, rank);
    out->basis = mat_new(rows, rank);
    memcpy(out->basis.a, vecs.a, rows * rank * sizeof(double));
    mat_free(&vecs);
    return OK;
  }
  mat m = unfold(t, mode);
  mat g = gram_t_from_cols(m.a, m.rows, m.cols);
  double* lambda = (double*)xcalloc(cols > 0 ? cols : 1, sizeof(double));
  mat vecs;
  int st = sym_eig_desc(&g, lambda, &vecs);
  mat_free(&g);
  if (st) { mat_free(&m); free(lambda); return st; }
  double smax = cols == 0 ? 0.0 : sqrt(lambda[0]);
  double floor_ = 1e-14 * smax;
  for (size_t i = 0; i < cols; ++i)
    if (sqrt(lambda[i]) <= floor_) lambda[i] = 0.0;
  size_t rank = truncation_rank(lambda, cols, delta);
  if (rank == (size_t)-1) { mat_free(&m); mat_free(&vecs); free(lambda); return EINVAL_; }
  out->discarded = trailing_sum(lambda, cols, rank);
  mat kept = mat_new(cols, rank);
  memcpy(kept.a, vecs.a, cols * rank * sizeof(double));
  out->basis = multiply(&m, &kept, 0, 0);
  for (size_t j = 0; j < rank; ++j) {
    double inv = 1.0 / sqrt(lambda[j]);
    double* bj = out->basis.a + j * rows;
    for (size_t i = 0; i < rows; ++i) bj[i] *= inv;
  }
  orthonormalize_columns(&out->basis);
  out->evals = (double*)xcalloc(rows, sizeof(double));
  out->n_evals = rows;
  for (size_t i = 0; i < cols; ++i) out->evals[i] = lambda[i];
  mat_free(&kept);
  mat_free(&m);
  mat_free(&vecs);
  free(lambda);
  return OK;
}

static void subspace_free(subspace* s) {
  mat_free(&s->basis);
  free(s->evals);
  s->evals = NULL;
}

/* ------------------------------------------------------------- ISVD state */
/* GrowableRowMatrix (isvd.hpp:18-60) kept as a dense row-major buffer with
 * a column capacity; the arithmetic (right_multiply, column_gram) follows
 * isvd.cpp:66-100 exactly. */
typedef struct {
  size_t rows, cols, cap_cols, cap_rows;
  double* a; /* row-major, stride cap_cols */
} growmat;

static void gm_reserve(growmat* g, size_t rows, size_t cols) {
  if (cols > g->cap_cols || rows > g->cap_rows) {
    size_t nc = cols > g->cap_cols ? cols + 8 : g->cap_cols;
    size_t nr = rows > g->cap_rows ? (rows * 2 + 16) : g->cap_rows;
    double* na = (double*)xcalloc(nr * nc, sizeof(double));
    for (size_t i = 0; i < g->rows; ++i)
      for (size_t j = 0; j < g->cols; ++j) na[i * nc + j] = g->a[i * g->cap_cols + j];
    free(g->a);
    g->a = na;
    g->cap_cols = nc;
    g->cap_rows = nr;
  }
}
static double* gm_row(growmat* g, size_t i) { return g->a + i * g->cap_cols; }

static void gm_append_row(growmat* g, const double* v) {
  gm_reserve(g, g->rows + 1, g->cols);
  double* r = gm_row(g, g->rows);
  for (size_t j = 0; j < g->cols; ++j) r[j] = v[j];
  g->rows++;
}
static void gm_append_zero_row(growmat* g) {
  gm_reserve(g, g->rows + 1, g->cols);
  double* r = gm_row(g, g->rows);
  for (size_t j = 0; j < g->cols; ++j) r[j] = 0.0;
  g->rows++;
}
/* right_multiply (isvd.cpp:66-84). */
static void gm_right_multiply(growmat* g, const mat* m) {
  size_t nc = m->cols, oc = g->cols;
  gm_reserve(g, g->rows, nc);
  double* tmp = (double*)xcalloc(nc, sizeof(double));
  for (size_t i = 0; i < g->rows; ++i) {
    double* row = gm_row(g, i);
    for (size_t j = 0; j < nc; ++j) {
      double s = 0.0;
      for (size_t l = 0; l < oc; ++l) s += row[l] * M(*m, l, j);
      tmp[j] = s;
    }
    memcpy(row, tmp, nc * sizeof(double));
    for (size_t j = nc; j < oc; ++j) row[j] = 0.0;
  }
  free(tmp);
  g->cols = nc;
}
/* column_gram (isvd.cpp:86-100). */
static mat gm_column_gram(growmat* g) {
  mat out = mat_new(g->cols, g->cols);
  for (size_t i = 0; i < g->rows; ++i) {
    const double* row = gm_row(g, i);
    for (size_t j = 0; j < g->cols; ++j) {
      double w = row[j];
      if (w == 0.0) continue;
      double* gj = out.a + j * g->cols;
      for (size_t l = 0; l <= j; ++l) gj[l] += row[l] * w;
    }
  }
  for (size_t j = 0; j < g->cols; ++j)
    for (size_t i = 0; i < j; ++i) M(out, j, i) = M(out, i, j);
  return out;
}

typedef struct {
  growmat left;
  double* sigma;
  size_t rank;
  mat right; /* n x r */
  double squared_error;
  size_t insertions;
  size_t reorthogonalize_every; /* ISVDOptions (isvd.hpp:62-67) */
} isvd_t;

/* GrowableRowMatrix::reorthogonalize (isvd.cpp:102-124): MGS over columns. */
static void gm_reorthogonalize(growmat* g) {
  for (size_t j = 0; j < g->cols; ++j) {
    for (size_t i = 0; i < j; ++i) {
      double dot = 0.0;
      for (size_t r = 0; r < g->rows; ++r) {
        const double* row = gm_row(g, r);
        dot += row[i] * row[j];
      }
      for (size_t r = 0; r < g->rows; ++r) {
        double* row = gm_row(g, r);
        row[j] -= dot * row[i];
      }
    }
    double sq = 0.0;
    for (size_t r = 0; r < g->rows; ++r) {
      const double v = gm_row(g, r)[j];
      sq += v * v;
    }
    const double norm = sqrt(sq);
    if (norm > 0.0)
      for (size_t r = 0; r < g->rows; ++r) gm_row(g, r)[j] /= norm;
  }
}

typedef struct { mat inner_left; size_t r_old, r_new; int degenerate; double added; } addrow_res;

/* add_row (isvd.cpp:163-250), with the optional periodic re-orthogonalization. */
static int add_row(isvd_t* st, const double* b, double abs_tol, addrow_res* res) {
  size_t n = st->right.rows, r = st->rank;
  memset(res, 0, sizeof *res);
  if (abs_tol < 0.0) { set_err("add_row: threshold must be nonnegative"); return EINVAL_; }
  double norm_b = sqrt(sumsq(b, n));
  double* p = (double*)xcalloc(r + 1, sizeof(double));
  double* e = (double*)xcalloc(n + 1, sizeof(double));
  memcpy(e, b, n * sizeof(double));
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t j = 0; j < r; ++j) {
      const double* qj = st->right.a + j * n;
      double dot = 0.0;
      for (size_t i = 0; i < n; ++i) dot += qj[i] * e[i];
      p[j] += dot;
      for (size_t i = 0; i < n; ++i) e[i] -= dot * qj[i];
    }
  }
  double k = sqrt(sumsq(e, n));
  res->r_old = r;
  res->degenerate = (k <= 1e-12 * norm_b);
  if (res->degenerate && r == 0) {
    gm_append_zero_row(&st->left);
    st->insertions++;
    res->inner_left = mat_new(1, 0);
    free(p); free(e);
    return OK;
  }
  size_t inner_cols = res->degenerate ? r : r + 1;
  mat sp = mat_new(r + 1, inner_cols);
  for (size_t j = 0; j < r; ++j) {
    M(sp, j, j) = st->sigma[j];
    M(sp, r, j) = p[j];
  }
  if (!res->degenerate) M(sp, r, r) = k;
  smallsvd inner;
  int stt = small_svd_truncated(&sp, abs_tol, &inner);
  mat_free(&sp);
  if (stt) { free(p); free(e); return stt; }
  res->r_new = inner.rank;
  res->added = inner.discarded;
  if (res->degenerate) res->added += k * k;
  st->squared_error += res->added;
  mat newright;
  if (res->degenerate) {
    newright = multiply(&st->right, &inner.right, 0, 0);
  } else {
    mat q = mat_new(n, 1);
    double inv = 1.0 / k;
    for (size_t i = 0; i < n; ++i) q.a[i] = e[i] * inv;
    mat h = hcat(&st->right, &q);
    newright = multiply(&h, &inner.right, 0, 0);
    mat_free(&h);
    mat_free(&q);
  }
  mat_free(&st->right);
  st->right = newright;
  mat top = mat_new(r, res->r_new);
  double* last = (double*)xcalloc(res->r_new + 1, sizeof(double));
  for (size_t j = 0; j < res->r_new; ++j) {
    for (size_t i = 0; i < r; ++i) M(top, i, j) = M(inner.left, i, j);
    last[j] = M(inner.left, r, j);
  }
  gm_right_multiply(&st->left, &top);
  gm_append_row(&st->left, last);
  free(st->sigma);
  st->sigma = inner.sigma;
  inner.sigma = NULL;
  st->rank = inner.rank;
  res->inner_left = inner.left;
  inner.left.a = NULL;
  st->insertions++;
  /* isvd.cpp:243-248 */
  if (st->reorthogonalize_every > 0 && st->insertions % st->reorthogonalize_every == 0) {
    gm_reorthogonalize(&st->left);
    orthonormalize_columns(&st->right);
  }
  mat_free(&top);
  free(last);
  mat_free(&inner.right);
  free(p);
  free(e);
  return OK;
}

/* -------------------------------------------------------- streaming state */
#define MAXMETRICS_INIT 64
struct orc_state {
  int order;              /* d */
  size_t n_d;
  double tau;
  ten core;               /* R_0..R_{d-1} */
  mat factors[MAXD];      /* k < d-1 */
  size_t slice_dims[MAXD];
  isvd_t isvd;
  ten v;                  /* same dims as core; buffer == isvd.right */
  double total_input_sq, nonstream_discarded_sq;
  orc_metrics* metrics;
  size_t n_metrics, cap_metrics;
};

static void push_metrics(orc_state* s, const orc_metrics* m) {
  if (s->n_metrics == s->cap_metrics) {
    s->cap_metrics = s->cap_metrics ? s->cap_metrics * 2 : MAXMETRICS_INIT;
    s->metrics = (orc_metrics*)realloc(s->metrics, s->cap_metrics * sizeof(orc_metrics));
  }
  s->metrics[s->n_metrics++] = *m;
}

/* check_core_coupling (streaming.cpp:39-64). */
static int check_core_coupling(const orc_state* s) {
  int d = s->order;
  size_t r = s->core.dims[d - 1];
  size_t slab = r == 0 ? 0 : s->core.size / r;
  double diff_sq = 0.0;
  for (size_t j = 0; j < r; ++j) {
    double sv = s->isvd.sigma[j];
    const double* c = s->core.a + j * slab;
    const double* v = s->v.a + j * slab;
    for (size_t i = 0; i < slab; ++i) {
      double diff = c[i] - v[i] * sv;
      diff_sq += diff * diff;
    }
  }
  double cn = ten_norm(&s->core);
  if (sqrt(diff_sq) > 1e-8 * cn + 1e-300) {
    set_err("streaming state invariant violated: core no longer matches the ISVD factorization");
    return EDRIFT;
  }
  return OK;
}

static double estimate(const orc_state* s) {
  if (s->total_input_sq <= 0.0) return 0.0;
  double booked = s->isvd.squared_error + s->nonstream_discarded_sq;
  return sqrt((booked > 0.0 ? booked : 0.0) / s->total_input_sq);
}

/* right_matrix_from_v (streaming.cpp:19-26): copy of the v buffer. */
static void refresh_right_from_v(orc_state* s) {
  int d = s->order;
  size_t r = s->v.dims[d - 1];
  size_t n = r == 0 ? 0 : s->v.size / r;
  mat_free(&s->isvd.right);
  s->isvd.right = mat_new(n, r);
  memcpy(s->isvd.right.a, s->v.a, s->v.size * sizeof(double));
}

static void state_free(orc_state* s) {
  if (!s) return;
  ten_free(&s->core);
  ten_free(&s->v);
  for (int k = 0; k < MAXD; ++k) mat_free(&s->factors[k]);
  free(s->isvd.left.a);
  free(s->isvd.sigma);
  mat_free(&s->isvd.right);
  free(s->metrics);
  free(s);
}
int tko_set_reorthogonalize_every(orc_state* s, int64_t k) {
  if (k < 0) { set_err("reorthogonalize_every must be nonnegative"); return EINVAL_; }
  s->isvd.reorthogonalize_every = (size_t)k;
  return OK;
}

void tko_destroy(orc_state* s) { state_free(s); }

/* isvd_init validation (isvd.cpp:135-161). */
static int isvd_init(isvd_t* st, const mat* left, double* sigma, size_t r,
                     const mat* right, double sq_err) {
  if (left->cols != r || right->cols != r) { set_err("isvd_init: factor widths must equal rank"); return EINVAL_; }
  if (orth_defect(left) > 1e-6) { set_err("isvd_init: left factor not orthonormal"); return EINVAL_; }
  if (orth_defect(right) > 1e-6) { set_err("isvd_init: right factor not orthonormal"); return EINVAL_; }
  for (size_t j = 0; j < r; ++j) {
    if (!(sigma[j] > 0.0)) { set_err("isvd_init: singular values must be positive"); return EINVAL_; }
    if (j > 0 && sigma[j] > sigma[j - 1]) { set_err("isvd_init: singular values must descend"); return EINVAL_; }
  }
  if (!(sq_err >= 0.0)) { set_err("isvd_init: initial squared error must be nonnegative"); return EINVAL_; }
  memset(st, 0, sizeof *st);
  st->left.cols = r;
  gm_reserve(&st->left, left->rows, r);
  for (size_t i = 0; i < left->rows; ++i) {
    double* row = gm_row(&st->left, i);
    for (size_t j = 0; j < r; ++j) row[j] = M(*left, i, j);
  }
  st->left.rows = left->rows;
  st->sigma = (double*)xcalloc(r + 1, sizeof(double));
  memcpy(st->sigma, sigma, r * sizeof(double));
  st->rank = r;
  st->right = mat_new(right->rows, right->cols);
  memcpy(st->right.a, right->a, right->rows * right->cols * sizeof(double));
  st->squared_error = sq_err;
  return OK;
}

/* sthosvd (sthosvd.cpp:94-133) + stream_init (streaming.cpp:83-124). */
int tko_stream_init(const double* x, int32_t order, const int64_t* dims,
                    double tau, orc_state** out) {
  *out = NULL;
  if (order < 2) { set_err("stream_init: need at least one non-streaming mode"); return EINVAL_; }
  if (order > MAXD) { set_err("stream_init: order exceeds %d", MAXD); return EINVAL_; }
  size_t dz[MAXD];
  for (int k = 0; k < order; ++k) dz[k] = (size_t)dims[k];
  ten xt = ten_new(order, dz);
  memcpy(xt.a, x, xt.size * sizeof(double));
  double norm = ten_norm(&xt);
  if (norm == 0.0) { ten_free(&xt); set_err("stream_init: initial batch must be nonzero to seed a factorization"); return EINVAL_; }
  if (!(tau > 0.0 && tau < 1.0)) { ten_free(&xt); set_err("sthosvd: tau must lie in (0, 1)"); return EINVAL_; }

  orc_state* s = (orc_state*)xcalloc(1, sizeof(orc_state));
  s->order = order;
  s->tau = tau;
  double delta = tau * norm / sqrt((double)order);
  ten core = ten_copy(&xt);
  double discarded = 0.0;
  double* last_evals = NULL;
  mat last_basis = {0, 0, NULL};
  for (int k = 0; k < order; ++k) {
    subspace sub;
    int st = mode_subspace(&core, k, delta, &sub);
    if (st) { ten_free(&core); ten_free(&xt); state_free(s); return st; }
    ten nc = ttm(&core, k, &sub.basis, 1);
    ten_free(&core);
    core = nc;
    discarded += sub.discarded;
    if (k == order - 1) {
      last_evals = sub.evals;
      sub.evals = NULL;
      last_basis = sub.basis;
      sub.basis.a = NULL;
    } else {
      s->factors[k] = sub.basis;
      sub.basis.a = NULL;
    }
    subspace_free(&sub);
  }
  int kd = order - 1;
  size_t r = core.dims[kd];
  double* sv = (double*)xcalloc(r + 1, sizeof(double));
  for (size_t j = 0; j < r; ++j) sv[j] = sqrt(last_evals[j]);
  ten v = ten_copy(&core);
  size_t slab = r == 0 ? 0 : v.size / r;
  for (size_t j = 0; j < r; ++j) {
    double inv = 1.0 / sv[j];
    double* p = v.a + j * slab;
    for (size_t i = 0; i < slab; ++i) p[i] *= inv;
  }
  mat right = mat_new(slab, r);
  memcpy(right.a, v.a, v.size * sizeof(double));
  int st = isvd_init(&s->isvd, &last_basis, sv, r, &right, discarded);
  free(sv);
  mat_free(&right);
  mat_free(&last_basis);
  free(last_evals);
  if (st) { ten_free(&core); ten_free(&v); ten_free(&xt); state_free(s); return st; }
  s->core = core;
  s->v = v;
  s->n_d = (size_t)dims[kd];
  for (int k = 0; k < kd; ++k) s->slice_dims[k] = (size_t)dims[k];
  s->total_input_sq = sumsq(xt.a, xt.size);
  ten_free(&xt);
  st = check_core_coupling(s);
  if (st) { state_free(s); return st; }
  *out = s;
  return OK;
}

/* process_nonstreaming_mode (streaming.cpp:126-155). y is replaced. */
static int process_mode(orc_state* s, ten* y, int mode, double delta,
                        double* res_norm, int* expanded) {
  const mat* u = &s->factors[mode];
  ten projected = ttm(y, mode, u, 1);
  ten residual = ttm(&projected, mode, u, 0);
  for (size_t i = 0; i < residual.size; ++i) residual.a[i] = y->a[i] - residual.a[i];
  double rn = ten_norm(&residual);
  *res_norm = rn;
  *expanded = 0;
  if (rn <= delta) {
    s->nonstream_discarded_sq += rn * rn;
    ten_free(y);
    *y = projected;
    ten_free(&residual);
    return OK;
  }
  subspace sub;
  int st = mode_subspace(&residual, mode, delta, &sub);
  if (st) { ten_free(&projected); ten_free(&residual); return st; }
  size_t grown = sub.basis.cols;
  ten carried = ttm(&residual, mode, &sub.basis, 1);
  mat nu = hcat(u, &sub.basis);
  mat_free(&s->factors[mode]);
  s->factors[mode] = nu;
  ten nc = pad_with_zeros(&s->core, mode, grown);
  ten_free(&s->core);
  s->core = nc;
  ten nv = pad_with_zeros(&s->v, mode, grown);
  ten_free(&s->v);
  s->v = nv;
  refresh_right_from_v(s);
  s->nonstream_discarded_sq += sub.discarded;
  ten ny = concat_along_mode(mode, &projected, &carried);
  ten_free(y);
  *y = ny;
  ten_free(&projected);
  ten_free(&carried);
  ten_free(&residual);
  subspace_free(&sub);
  *expanded = 1;
  return OK;
}

/* stream_update (streaming.cpp:157-233). */
int tko_stream_update(orc_state* s, const double* yin) {
  int d = s->order;
  orc_metrics rec;
  memset(&rec, 0, sizeof rec);
  rec.slice_index = (int64_t)s->n_d;
  ten y = ten_new(d - 1, s->slice_dims);
  memcpy(y.a, yin, y.size * sizeof(double));
  rec.slice_norm = ten_norm(&y);
  s->total_input_sq += rec.slice_norm * rec.slice_norm;
  if (rec.slice_norm == 0.0) {
    gm_append_zero_row(&s->isvd.left);
    s->n_d++;
    for (int k = 0; k < d; ++k) rec.ranks[k] = (int64_t)s->core.dims[k];
    rec.ranks[d - 1] = (int64_t)s->isvd.rank;
    rec.error_estimate = estimate(s);
    push_metrics(s, &rec);
    ten_free(&y);
    return OK;
  }
  double delta = s->tau * rec.slice_norm / sqrt((double)d);
  for (int k = 0; k + 1 < d; ++k) {
    int expanded;
    int st = process_mode(s, &y, k, delta, &rec.mode_residuals[k], &expanded);
    if (st) { ten_free(&y); return st; }
    if (expanded) rec.expanded_mask |= 1 << k;
  }
  rec.projected_norm = ten_norm(&y);

  mat p_gram = gm_column_gram(&s->isvd.left);
  addrow_res ins;
  int st = add_row(&s->isvd, y.a, delta, &ins);
  if (st) { mat_free(&p_gram); ten_free(&y); return st; }
  mat top = mat_new(ins.r_old, ins.r_new);
  for (size_t j = 0; j < ins.r_new; ++j)
    for (size_t i = 0; i < ins.r_old; ++i) M(top, i, j) = M(ins.inner_left, i, j);
  mat rot = multiply(&top, &p_gram, 1, 0);
  ten newcore = ttm(&s->core, d - 1, &rot, 0);
  size_t slab = y.size;
  for (size_t j = 0; j < ins.r_new; ++j) {
    double w = M(ins.inner_left, ins.r_old, j);
    if (w == 0.0) continue;
    double* c = newcore.a + j * slab;
    for (size_t i = 0; i < slab; ++i) c[i] += w * y.a[i];
  }
  ten_free(&s->core);
  s->core = newcore;
  /* v_from_right_matrix (streaming.cpp:28-35, 221-222) */
  ten_free(&s->v);
  s->v = ten_new(d, s->core.dims);
  memcpy(s->v.a, s->isvd.right.a, s->v.size * sizeof(double));
  s->n_d++;
  mat_free(&top);
  mat_free(&rot);
  mat_free(&p_gram);
  mat_free(&ins.inner_left);
  ten_free(&y);
  st = check_core_coupling(s);
  for (int k = 0; k < d; ++k) rec.ranks[k] = (int64_t)s->core.dims[k];
  rec.error_estimate = estimate(s);
  if (st) return st;
  push_metrics(s, &rec);
  return OK;
}

int tko_process_mode(orc_state* s, const double* yin, const int64_t* ydims,
                     int32_t mode, double delta, double* y_out,
                     int64_t y_out_cap, int64_t* ydims_out, double* res) {
  int d = s->order;
  if (mode < 0 || mode >= d - 1) { set_err("process_mode: mode out of range"); return EINVAL_; }
  size_t dz[MAXD];
  for (int k = 0; k < d - 1; ++k) dz[k] = (size_t)ydims[k];
  if (dz[mode] != s->factors[mode].rows) { set_err("process_mode: shape mismatch"); return EINVAL_; }
  ten y = ten_new(d - 1, dz);
  memcpy(y.a, yin, y.size * sizeof(double));
  int expanded;
  int st = process_mode(s, &y, mode, delta, res, &expanded);
  if (st) { ten_free(&y); return st; }
  if ((int64_t)y.size > y_out_cap) { ten_free(&y); set_err("process_mode: output capacity"); return EINVAL_; }
  memcpy(y_out, y.a, y.size * sizeof(double));
  for (int k = 0; k < d - 1; ++k) ydims_out[k] = (int64_t)y.dims[k];
  ten_free(&y);
  return OK;
}

int tko_query(const orc_state* s, orc_dims* o) {
  memset(o, 0, sizeof *o);
  o->order = s->order;
  o->n_d = (int64_t)s->n_d;
  o->rank = (int64_t)s->isvd.rank;
  o->insertions = (int64_t)s->isvd.insertions;
  for (int k = 0; k < s->order; ++k) o->core_dims[k] = (int64_t)s->core.dims[k];
  for (int k = 0; k + 1 < s->order; ++k) o->slice_dims[k] = (int64_t)s->slice_dims[k];
  o->tau = s->tau;
  o->squared_error = s->isvd.squared_error;
  o->total_input_sq = s->total_input_sq;
  o->nonstream_discarded_sq = s->nonstream_discarded_sq;
  return OK;
}

int tko_export_state(const orc_state* s, double* core, double* factors,
                     double* sigma, double* left, double* right) {
  if (core) memcpy(core, s->core.a, s->core.size * sizeof(double));
  if (factors) {
    size_t off = 0;
    for (int k = 0; k + 1 < s->order; ++k) {
      size_t sz = s->factors[k].rows * s->factors[k].cols;
      memcpy(factors + off, s->factors[k].a, sz * sizeof(double));
      off += sz;
    }
  }
  if (sigma) memcpy(sigma, s->isvd.sigma, s->isvd.rank * sizeof(double));
  if (left) {
    const growmat* g = &s->isvd.left;
    for (size_t i = 0; i < g->rows; ++i)
      for (size_t j = 0; j < g->cols; ++j)
        left[j * g->rows + i] = g->a[i * g->cap_cols + j];
  }
  if (right)
    memcpy(right, s->isvd.right.a, s->isvd.right.rows * s->isvd.right.cols * sizeof(double));
  return OK;
}

int tko_last_metrics(const orc_state* s, orc_metrics* out) {
  if (s->n_metrics == 0) { set_err("no metrics recorded"); return EINVAL_; }
  *out = s->metrics[s->n_metrics - 1];
  return OK;
}
int64_t tko_metrics_count(const orc_state* s) { return (int64_t)s->n_metrics; }
int tko_metrics_at(const orc_state* s, int64_t i, orc_metrics* out) {
  if (i < 0 || (size_t)i >= s->n_metrics) { set_err("metrics index out of range"); return EINVAL_; }
  *out = s->metrics[i];
  return OK;
}

/* assemble_streaming_state (streaming.cpp:242-263). */
int tko_assemble(const orc_dims* dm, const double* core, const double* factors,
                 const double* sigma, const double* left, const double* right,
                 orc_state** out) {
  *out = NULL;
  int d = dm->order;
  if (d < 2 || d > MAXD) { set_err("assemble_streaming_state: need d >= 2"); return EINVAL_; }
  orc_state* s = (orc_state*)xcalloc(1, sizeof(orc_state));
  s->order = d;
  s->tau = dm->tau;
  size_t cd[MAXD];
  for (int k = 0; k < d; ++k) cd[k] = (size_t)dm->core_dims[k];
  s->core = ten_new(d, cd);
  memcpy(s->core.a, core, s->core.size * sizeof(double));
  size_t off = 0;
  for (int k = 0; k + 1 < d; ++k) {
    s->slice_dims[k] = (size_t)dm->slice_dims[k];
    s->factors[k] = mat_new(s->slice_dims[k], cd[k]);
    memcpy(s->factors[k].a, factors + off, s->slice_dims[k] * cd[k] * sizeof(double));
    off += s->slice_dims[k] * cd[k];
  }
  size_t r = cd[d - 1];
  size_t n = r == 0 ? 0 : s->core.size / r;
  s->isvd.rank = r;
  s->isvd.sigma = (double*)xcalloc(r + 1, sizeof(double));
  memcpy(s->isvd.sigma, sigma, r * sizeof(double));
  s->isvd.left.cols = r;
  gm_reserve(&s->isvd.left, (size_t)dm->n_d, r);
  for (size_t i = 0; i < (size_t)dm->n_d; ++i)
    for (size_t j = 0; j < r; ++j) gm_row(&s->isvd.left, i)[j] = left[j * dm->n_d + i];
  s->isvd.left.rows = (size_t)dm->n_d;
  s->isvd.right = mat_new(n, r);
  memcpy(s->isvd.right.a, right, n * r * sizeof(double));
  s->isvd.squared_error = dm->squared_error;
  s->isvd.insertions = (size_t)dm->insertions;
  s->n_d = (size_t)dm->n_d;
  s->total_input_sq = dm->total_input_sq;
  s->nonstream_discarded_sq = dm->nonstream_discarded_sq;
  s->v = ten_new(d, cd);
  memcpy(s->v.a, right, s->v.size * sizeof(double));
  int st = check_core_coupling(s);
  if (st) { state_free(s); return st; }
  *out = s;
  return OK;
}

/* ---------------------------------------------------- building-block ABI */
int tko_sym_eig_desc(int64_t n, const double* g, double* evals, double* evecs) {
  mat gm = {(size_t)n, (size_t)n, (double*)g};
  mat v;
  int st = sym_eig_desc(&gm, evals, &v);
  if (st) return st;
  memcpy(evecs, v.a, (size_t)(n * n) * sizeof(double));
  mat_free(&v);
  return OK;
}

int64_t tko_truncation_rank(int64_t n, const double* evals, double delta) {
  size_t r = truncation_rank(evals, (size_t)n, delta);
  return r == (size_t)-1 ? -1 : (int64_t)r;
}

int tko_small_svd_truncated(int64_t m, int64_t n, const double* a, double thr,
                            double* left, double* sigma, double* right,
                            int64_t* rank, double* disc) {
  mat am = {(size_t)m, (size_t)n, (double*)a};
  smallsvd s;
  int st = small_svd_truncated(&am, thr, &s);
  if (st) return st;
  *rank = (int64_t)s.rank;
  *disc = s.discarded;
  memcpy(left, s.left.a, (size_t)m * s.rank * sizeof(double));
  memcpy(sigma, s.sigma, s.rank * sizeof(double));
  memcpy(right, s.right.a, (size_t)n * s.rank * sizeof(double));
  smallsvd_free(&s);
  return OK;
}

int tko_mode_subspace(const double* t, int32_t order, const int64_t* dims,
                      int32_t mode, double delta, double* basis, int64_t* rank,
                      double* evals, double* disc) {
  size_t dz[MAXD];
  for (int k = 0; k < order; ++k) dz[k] = (size_t)dims[k];
  ten tt = ten_new(order, dz);
  memcpy(tt.a, t, tt.size * sizeof(double));
  subspace sub;
  int st = mode_subspace(&tt, mode, delta, &sub);
  ten_free(&tt);
  if (st) return st;
  *rank = (int64_t)sub.basis.cols;
  *disc = sub.discarded;
  memcpy(basis, sub.basis.a, sub.basis.rows * sub.basis.cols * sizeof(double));
  memcpy(evals, sub.evals, sub.n_evals * sizeof(double));
  subspace_free(&sub);
  return OK;
}

int tko_ttm(const double* t, int32_t order, const int64_t* dims, int32_t mode,
            const double* a, int64_t a_rows, int64_t a_cols,
            int32_t transpose_a, double* out) {
  size_t dz[MAXD];
  for (int k = 0; k < order; ++k) dz[k] = (size_t)dims[k];
  ten tt = {order, {0}, 1, (double*)t};
  for (int k = 0; k < order; ++k) { tt.dims[k] = dz[k]; tt.size *= dz[k]; }
  size_t contracted = transpose_a ? (size_t)a_rows : (size_t)a_cols;
  if (contracted != dz[mode]) { set_err("ttm: matrix does not match mode size"); return EINVAL_; }
  mat am = {(size_t)a_rows, (size_t)a_cols, (double*)a};
  ten o = ttm(&tt, mode, &am, transpose_a);
  memcpy(out, o.a, o.size * sizeof(double));
  ten_free(&o);
  return OK;
}
