/*
 * rpc_oracle.c — CPU restatement of the reference accelerated RPCholesky path.
 *
 * TEST INFRASTRUCTURE ONLY (see rpc_oracle.h).  Every function cites the
 * reference definition it restates (paths relative to
 * /root/reference/proj/include/rpchol/).  Arithmetic follows the reference's
 * effective build: IEEE binary64, no contraction into FMA (-ffp-contract=off;
 * the reference Release build has no -march, i.e. SSE2 without FMA).  Dot
 * products and reductions are evaluated in ascending index order; the
 * reference delegates those to Eigen 3.4, whose blocking order is not
 * reproducible without its sources, so agreement there is to rounding (see
 * DESIGN.md §3 "parity pins").
 *
 * Row-parallel loops (OpenMP) never change any element's summation order, so
 * results are bit-identical for every thread count — the same invariant the
 * reference states for KernelOracle (oracle.hpp:176-178).
 */
#include "rpc_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* rpo_last_error(void) { return g_err; }

/* Releases one buffer a result handed over (a factor kept without copying). */
void rpo_free(void* p) { free(p); }

/* ---- rng.hpp:27-42  SplitMix64::next_u64 / next_double --------------- */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* The n-th (0-based) next_u64() of SplitMix64(seed): state advances by the
 * golden-ratio increment before mixing (rng.hpp:31-36). */
uint64_t rpo_splitmix64_draw(uint64_t seed, uint64_t n) {
  return mix64(seed + (n + 1) * 0x9e3779b97f4a7c15ULL);
}

/* rng.hpp:40-42 */
double rpo_u01(uint64_t z) { return (double)(z >> 11) * 0x1.0p-53; }

/* ---- rng.hpp:67-75  cumulative_sums: sequential inclusive scan ------- */
void rpo_cumulative_sums(const double* w, int64_t n, double* out) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += w[i];
    out[i] = acc;
  }
}

/* ---- decision-margin recorder (instrumentation for the parity tests) --
 * Not part of the reference: records how far each random decision was from
 * flipping, so a pivot match between two implementations whose sums differ
 * only by association can be shown to be robust rather than lucky.
 *   draw margin  = min(target - cumsum[i-1], cumsum[i] - target) / total
 *                  (distance of the target to the nearer bucket edge)
 *   sweep margin = |u_i * r - h_ii| / u_i   (rpcholesky.hpp:179 accept test)
 * Off by default; rpo_margins_reset() turns it on and clears the minima. */
static int g_margins_on;
static double g_min_draw = 1.0 / 0.0, g_min_sweep = 1.0 / 0.0;
static int64_t g_n_draws, g_n_decisions;

void rpo_margins_reset(int on) {
  g_margins_on = on;
  g_min_draw = g_min_sweep = 1.0 / 0.0;
  g_n_draws = g_n_decisions = 0;
}

void rpo_margins_get(double* min_draw, double* min_sweep, int64_t* n_draws, int64_t* n_decisions) {
  *min_draw = g_min_draw;
  *min_sweep = g_min_sweep;
  *n_draws = g_n_draws;
  *n_decisions = g_n_decisions;
}

/* ---- rng.hpp:80-96  sample_discrete ---------------------------------- */
int rpo_sample_discrete(const double* cumsum, int64_t n, double u01, int64_t* idx) {
  if (n == 0) return fail(RPO_EINVAL, "sample_discrete: empty weights");
  const double total = cumsum[n - 1];
  if (!(total > 0.0)) return fail(RPO_EINVAL, "sample_discrete: total weight must be > 0");
  const double target = u01 * total;
  /* std::upper_bound: first element > target */
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (target < cumsum[mid]) hi = mid; else lo = mid + 1;
  }
  int64_t i = lo;
  if (i >= n) i = n - 1;
  while (i > 0 && cumsum[i] == cumsum[i - 1]) --i;
  *idx = i;
  if (g_margins_on) {
    const double below = target - (i > 0 ? cumsum[i - 1] : 0.0), above = cumsum[i] - target;
    const double mg = (below < above ? below : above) / total;
    if (mg < g_min_draw) g_min_draw = mg;
    ++g_n_draws;
  }
  return RPO_OK;
}

/* ---- oracle.hpp:243-258  KernelOracle ctor; 195-207 DenseOracle ctor -- */
int rpo_oracle_kernel(rpo_oracle* o, const double* x, int64_t n, int64_t d, int kind,
                      double sigma, int dist_mode, int n_threads) {
  memset(o, 0, sizeof *o);
  /* data_matrix.hpp:22-29 */
  if (n < 1 || d < 1) return fail(RPO_EINVAL, "DataMatrix: need at least one point and one dimension");
  for (int64_t i = 0; i < n * d; ++i)
    if (!isfinite(x[i])) return fail(RPO_EINVAL, "DataMatrix: non-finite entry");
  /* kernels.hpp:47-49 */
  if (!(sigma > 0.0) || !isfinite(sigma)) return fail(RPO_EINVAL, "KernelSpec: bandwidth must be positive");
  if (kind < RPO_KERNEL_GAUSSIAN || kind > RPO_KERNEL_MATERN52)
    return fail(RPO_EINVAL, "unknown kernel kind");
  /* oracle.hpp:253-257 */
  if (dist_mode == RPO_DIST_GRAM && kind == RPO_KERNEL_L1LAPLACE)
    return fail(RPO_EINVAL, "KernelOracle: GramTrick requires an l2 translation-invariant kernel");
  o->is_dense = 0;
  o->n = n;
  o->x = x;
  o->d = d;
  o->kind = kind;
  o->sigma = sigma;
  o->dist_mode = dist_mode;
  o->n_threads = n_threads < 1 ? 1 : n_threads;
  o->sq_norms = (double*)malloc(sizeof(double) * (size_t)n);
  if (!o->sq_norms) return fail(RPO_ENOMEM, "out of memory");
  /* oracle.hpp:252  rowwise().squaredNorm() */
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double v = x[c * n + i];
      s += v * v;
    }
    o->sq_norms[i] = s;
  }
  return RPO_OK;
}

int rpo_oracle_dense(rpo_oracle* o, const double* a, int64_t n) {
  memset(o, 0, sizeof *o);
  for (int64_t i = 0; i < n * n; ++i)
    if (!isfinite(a[i])) return fail(RPO_EINVAL, "DenseOracle: non-finite entry");
  for (int64_t i = 0; i < n; ++i)
    if (a[i * n + i] < 0.0) return fail(RPO_EINVAL, "DenseOracle: negative diagonal entry");
  o->is_dense = 1;
  o->n = n;
  o->a = a;
  o->n_threads = 1;
  return RPO_OK;
}

void rpo_oracle_free(rpo_oracle* o) {
  free(o->sq_norms);
  o->sq_norms = NULL;
}

/* oracle.hpp:44-50 */
static int check_indices(const int64_t* idx, int64_t k, int64_t n, const char* what) {
  for (int64_t i = 0; i < k; ++i)
    if (idx[i] < 0 || idx[i] >= n) return fail(RPO_ERANGE, "%s: index out of range", what);
  return RPO_OK;
}

/* kernels.hpp:59-79  kernel_from_sq_dist (l2 kernels) */
static inline double kernel_from_sq(int kind, double sq, double sigma) {
  if (kind == RPO_KERNEL_MATERN32) {
    const double rho = sqrt(sq) / sigma;
    const double z = sqrt(3.0) * rho;
    return (1.0 + z) * exp(-z);
  }
  if (kind == RPO_KERNEL_MATERN52) {
    const double rho2 = sq / (sigma * sigma);
    const double z = sqrt(5.0 * rho2);
    return (1.0 + z + (5.0 / 3.0) * rho2) * exp(-z);
  }
  return exp(-0.5 * sq / (sigma * sigma));
}

/* KernelOracle::submatrix oracle.hpp:267-289 -> panel_block 296-320.
 * Column j of `out` (nr rows) for column point cols[j]. */
static void kernel_column(const rpo_oracle* o, const int64_t* rows, int64_t nr, int64_t col,
                          double* out) {
  const int64_t n = o->n, d = o->d;
  const double* x = o->x;
  if (o->kind == RPO_KERNEL_L1LAPLACE) {
    /* oracle.hpp:103-112 l1_dist_direct, then (-d / sigma).exp() (303) */
    for (int64_t a = 0; a < nr; ++a) out[a] = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double xc = x[c * n + col];
      const double* xr = x + c * n;
      for (int64_t a = 0; a < nr; ++a) out[a] += fabs(xr[rows[a]] - xc);
    }
    for (int64_t a = 0; a < nr; ++a) out[a] = exp(-out[a] / o->sigma);
    return;
  }
  if (o->dist_mode == RPO_DIST_DIRECT) {
    /* oracle.hpp:92-101 sq_dist_direct */
    for (int64_t a = 0; a < nr; ++a) out[a] = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double xc = x[c * n + col];
      const double* xr = x + c * n;
      for (int64_t a = 0; a < nr; ++a) {
        const double t = xr[rows[a]] - xc;
        out[a] += t * t;
      }
    }
  } else {
    /* oracle.hpp:71-90 sq_dist_gram: D = ((-2 xr.xc) + sqn_r) + sqn_c,
     * clamp at 0, pin equal global indices to 0. */
    for (int64_t a = 0; a < nr; ++a) out[a] = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double xc = x[c * n + col];
      const double* xr = x + c * n;
      for (int64_t a = 0; a < nr; ++a) out[a] += xr[rows[a]] * xc;
    }
    const double sqc = o->sq_norms[col];
    for (int64_t a = 0; a < nr; ++a) {
      double dd = (-2.0 * out[a] + o->sq_norms[rows[a]]) + sqc;
      if (dd < 0.0) dd = 0.0; /* cwiseMax(0.0) */
      if (rows[a] == col) dd = 0.0;
      out[a] = dd;
    }
  }
  for (int64_t a = 0; a < nr; ++a) out[a] = kernel_from_sq(o->kind, out[a], o->sigma);
}

int rpo_submatrix(const rpo_oracle* o, const int64_t* rows, int64_t nr, const int64_t* cols,
                  int64_t nc, double* out) {
  int rc;
  if ((rc = check_indices(rows, nr, o->n, o->is_dense ? "DenseOracle rows" : "KernelOracle rows")))
    return rc;
  if ((rc = check_indices(cols, nc, o->n, o->is_dense ? "DenseOracle cols" : "KernelOracle cols")))
    return rc;
  if (o->is_dense) {
    /* oracle.hpp:212-224 */
    for (int64_t j = 0; j < nc; ++j)
      for (int64_t i = 0; i < nr; ++i) out[j * nr + i] = o->a[cols[j] * o->n + rows[i]];
    return RPO_OK;
  }
#pragma omp parallel for schedule(static) num_threads(o->n_threads) if (nr * nc > 65536)
  for (int64_t j = 0; j < nc; ++j) kernel_column(o, rows, nr, cols[j], out + j * nr);
  return RPO_OK;
}

/* A(:, cols) for the full row range — PsdOracle::columns (oracle.hpp:188-191).
 * Row-blocked so that threads split rows; element order unchanged. */
static void oracle_columns(const rpo_oracle* o, const int64_t* cols, int64_t nc, double* g) {
  const int64_t n = o->n;
  if (o->is_dense) {
    for (int64_t j = 0; j < nc; ++j) memcpy(g + j * n, o->a + cols[j] * n, sizeof(double) * n);
    return;
  }
  const int64_t RB = 512;
  const int64_t nblk = (n + RB - 1) / RB;
#pragma omp parallel num_threads(o->n_threads)
  {
    int64_t rows[512];
    double tmp[512];
#pragma omp for schedule(static)
    for (int64_t blk = 0; blk < nblk; ++blk) {
      const int64_t r0 = blk * RB;
      const int64_t nr = (r0 + RB <= n) ? RB : n - r0;
      for (int64_t a = 0; a < nr; ++a) rows[a] = r0 + a;
      for (int64_t j = 0; j < nc; ++j) {
        kernel_column(o, rows, nr, cols[j], tmp);
        memcpy(g + j * n + r0, tmp, sizeof(double) * nr);
      }
    }
  }
}

/* ---- rpcholesky.hpp:167-201  rejection_sample_submatrix ------------- */
int rpo_rejection_sweep(double* h, int64_t b, const int64_t* proposals, uint64_t seed,
                        uint64_t draw0, int64_t* accepted, int64_t* positions, int64_t* m_out,
                        double* chol) {
  double* u = (double*)malloc(sizeof(double) * (size_t)b);
  double* l = (double*)calloc((size_t)(b * b), sizeof(double));
  if (!u || !l) {
    free(u);
    free(l);
    return fail(RPO_ENOMEM, "out of memory");
  }
  for (int64_t i = 0; i < b; ++i) u[i] = h[i * b + i];
  int64_t m = 0;
  for (int64_t i = 0; i < b; ++i) {
    const double r = rpo_u01(rpo_splitmix64_draw(seed, draw0 + (uint64_t)i));
    if (g_margins_on && u[i] > 0.0) {
      const double mg = fabs(u[i] * r - h[i * b + i]) / u[i];
      if (mg < g_min_sweep) g_min_sweep = mg;
      ++g_n_decisions;
    }
    if (u[i] * r < h[i * b + i]) {
      const double root = sqrt(h[i * b + i]);
      for (int64_t j = i; j < b; ++j) l[i * b + j] = h[i * b + j] / root;
      /* h(i+1:, i+1:) -= l l^T over the full trailing square (Eigen outer
       * product: each entry h_pq - (l_p * l_q), two roundings). */
      for (int64_t q = i + 1; q < b; ++q) {
        const double lq = l[i * b + q];
        for (int64_t p = i + 1; p < b; ++p) h[q * b + p] -= l[i * b + p] * lq;
      }
      positions[m] = i;
      accepted[m] = proposals[i];
      ++m;
    }
  }
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i) chol[j * m + i] = l[positions[j] * b + positions[i]];
  *m_out = m;
  free(u);
  free(l);
  return RPO_OK;
}

/* ---- rpcholesky.hpp:378-383  g -= F(:, :kcur) F(S, :kcur)^T --------- */
static void residual_gemm(const double* f, int64_t n, int64_t kcur, const double* fr, int64_t m,
                          double* g, int nthreads) {
  const int64_t IB = 64, JB = 4;
  const int64_t nblk = (n + IB - 1) / IB;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t i0 = blk * IB;
    const int64_t ni = (i0 + IB <= n) ? IB : n - i0;
    double acc[4][64];
    for (int64_t j0 = 0; j0 < m; j0 += JB) {
      const int64_t nj = (j0 + JB <= m) ? JB : m - j0;
      for (int64_t jj = 0; jj < JB; ++jj)
        for (int64_t ii = 0; ii < IB; ++ii) acc[jj][ii] = 0.0;
      for (int64_t k = 0; k < kcur; ++k) {
        const double* fc = f + k * n + i0;
        for (int64_t jj = 0; jj < nj; ++jj) {
          const double s = fr[k * m + j0 + jj];
          for (int64_t ii = 0; ii < ni; ++ii) acc[jj][ii] += fc[ii] * s;
        }
      }
      for (int64_t jj = 0; jj < nj; ++jj)
        for (int64_t ii = 0; ii < ni; ++ii) g[(j0 + jj) * n + i0 + ii] -= acc[jj][ii];
    }
  }
}

/* ---- rpcholesky.hpp:147-151  right_solve_lower_transposed: g <- g L^{-T}.
 * Row-wise forward substitution, ascending column order. */
static void right_solve_lt(const double* l, int64_t m, double* g, int64_t n, int nthreads) {
  const int64_t IB = 256;
  const int64_t nblk = (n + IB - 1) / IB;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t i0 = blk * IB;
    const int64_t ni = (i0 + IB <= n) ? IB : n - i0;
    for (int64_t j = 0; j < m; ++j) {
      double* gj = g + j * n + i0;
      for (int64_t q = 0; q < j; ++q) {
        const double ljq = l[q * m + j];
        const double* gq = g + q * n + i0;
        for (int64_t ii = 0; ii < ni; ++ii) gj[ii] -= gq[ii] * ljq;
      }
      const double ljj = l[j * m + j];
      for (int64_t ii = 0; ii < ni; ++ii) gj[ii] /= ljj;
    }
  }
}

static void diag_of(const rpo_oracle* o, double* u) {
  if (o->is_dense) {
    for (int64_t i = 0; i < o->n; ++i) u[i] = o->a[i * o->n + i];
  } else {
    /* oracle.hpp:262-265: kappa(x, x) = 1 */
    for (int64_t i = 0; i < o->n; ++i) u[i] = 1.0;
  }
}

/* rpcholesky.hpp:250-254 */
static int run_finished(const rpo_run_config* cfg, int64_t round, int64_t kcur) {
  if (cfg->mode == RPO_MODE_FIXED_ROUNDS) return round >= cfg->rounds;
  return kcur >= cfg->target_rank;
}

/* ---- rpcholesky.hpp:338-401  accelerated_rpcholesky ----------------- */
int rpo_accelerated_rpcholesky_bounded(const rpo_oracle* o, const rpo_run_config* cfg,
                                       int64_t max_rounds, rpo_result* res) {
  memset(res, 0, sizeof *res);
  const int64_t n = o->n;
  const int64_t b = cfg->block_size;
  const int nt = o->n_threads;
  if (b < 1) return fail(RPO_EINVAL, "accelerated_rpcholesky: block size must be >= 1");
  /* RunConfig factories reject t, k, b < 1 (rpcholesky.hpp:53, 64) */
  if (cfg->mode == RPO_MODE_FIXED_ROUNDS && cfg->rounds < 1)
    return fail(RPO_EINVAL, "RunConfig: t, b must be >= 1");
  if (cfg->mode == RPO_MODE_UNTIL_RANK && cfg->target_rank < 1)
    return fail(RPO_EINVAL, "RunConfig: k, b must be >= 1");
  double* u = (double*)malloc(sizeof(double) * (size_t)n);
  double* cumsum = (double*)malloc(sizeof(double) * (size_t)n);
  if (!u || !cumsum) {
    free(u);
    free(cumsum);
    return fail(RPO_ENOMEM, "out of memory");
  }
  diag_of(o, u);
  double trace_a = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (u[i] < 0.0) u[i] = 0.0; /* cwiseMax(0.0) == std::max */
    trace_a += u[i];
  }
  if (!(trace_a > 0.0)) {
    free(u);
    free(cumsum);
    return fail(RPO_EINVAL, "accelerated_rpcholesky: trace must be > 0");
  }
  int64_t cap = cfg->mode == RPO_MODE_FIXED_ROUNDS ? cfg->rounds * b : cfg->target_rank + b;
  if (cap > n) cap = n;
  double* f = (double*)malloc(sizeof(double) * (size_t)n * (size_t)cap);
  int64_t* pivots = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t* proposed = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  double* h = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* fr = (double*)malloc(sizeof(double) * (size_t)(b * (cap > 0 ? cap : 1)));
  int64_t* acc_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  int64_t* acc_pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  double* lsel = (double*)malloc(sizeof(double) * (size_t)(b * b));
  int64_t rounds_cap = 16;
  int64_t* all_prop = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rounds_cap * b));
  int64_t* all_cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)rounds_cap);
  int rc = RPO_OK;
  if (!f || !pivots || !proposed || !h || !fr || !acc_ids || !acc_pos || !lsel || !all_prop ||
      !all_cnt) {
    rc = fail(RPO_ENOMEM, "out of memory");
    goto done;
  }
  int64_t kcur = 0;
  double captured_sq = 0.0;
  uint64_t draw = 0;
  int64_t round;
  for (round = 0; !run_finished(cfg, round, kcur); ++round) {
    if (max_rounds >= 0 && round >= max_rounds) break;
    double usum = 0.0;
    for (int64_t i = 0; i < n; ++i) usum += u[i];
    if (!(usum > 0.0)) { /* rpcholesky.hpp:356-359 */
      res->rank_exhausted = 1;
      break;
    }
    if (cfg->stop_tol > 0.0 && (trace_a - captured_sq) <= cfg->stop_tol * trace_a) break;
    rpo_cumulative_sums(u, n, cumsum);
    for (int64_t j = 0; j < b; ++j) {
      rc = rpo_sample_discrete(cumsum, n, rpo_u01(rpo_splitmix64_draw(cfg->seed, draw++)),
                               &proposed[j]);
      if (rc) goto done;
    }
    /* H = A(S', S') - F(S', :) F(S', :)^T  (rpcholesky.hpp:366-371) */
    if ((rc = rpo_submatrix(o, proposed, b, proposed, b, h))) goto done;
    if (kcur > 0) {
      for (int64_t k = 0; k < kcur; ++k)
        for (int64_t i = 0; i < b; ++i) fr[k * b + i] = f[k * n + proposed[i]];
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < b; ++i) {
          double s = 0.0;
          for (int64_t k = 0; k < kcur; ++k) s += fr[k * b + i] * fr[k * b + j];
          h[j * b + i] -= s;
        }
    }
    int64_t m = 0;
    if ((rc = rpo_rejection_sweep(h, b, proposed, cfg->seed, draw, acc_ids, acc_pos, &m, lsel)))
      goto done;
    draw += (uint64_t)b;
    if (m > 0) {
      if (kcur + m > cap) {
        /* conservativeResize (rpcholesky.hpp:375-377) */
        const int64_t ncap = kcur + m;
        double* nf = (double*)realloc(f, sizeof(double) * (size_t)n * (size_t)ncap);
        int64_t* np = (int64_t*)realloc(pivots, sizeof(int64_t) * (size_t)ncap);
        double* nfr = (double*)realloc(fr, sizeof(double) * (size_t)(b * ncap));
        if (!nf || !np || !nfr) {
          rc = fail(RPO_ENOMEM, "out of memory");
          goto done;
        }
        f = nf;
        pivots = np;
        fr = nfr;
        cap = ncap;
      }
      double* g = f + kcur * n; /* new columns are written in place */
      oracle_columns(o, acc_ids, m, g);
      if (kcur > 0) {
        for (int64_t k = 0; k < kcur; ++k)
          for (int64_t i = 0; i < m; ++i) fr[k * m + i] = f[k * n + acc_ids[i]];
        residual_gemm(f, n, kcur, fr, m, g, nt);
      }
      right_solve_lt(lsel, m, g, n, nt);
      /* u -= rowwise ||g||^2; u = max(u, 0); captured_sq += ||g||_F^2 */
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < m; ++j) s += g[j * n + i] * g[j * n + i];
        u[i] -= s;
      }
      for (int64_t i = 0; i < n; ++i)
        if (u[i] < 0.0) u[i] = 0.0;
      double gs = 0.0;
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < n; ++i) gs += g[j * n + i] * g[j * n + i];
      captured_sq += gs;
      for (int64_t j = 0; j < m; ++j) pivots[kcur + j] = acc_ids[j];
      kcur += m;
    }
    if (round >= rounds_cap) {
      rounds_cap *= 2;
      int64_t* np = (int64_t*)realloc(all_prop, sizeof(int64_t) * (size_t)(rounds_cap * b));
      int64_t* nc = (int64_t*)realloc(all_cnt, sizeof(int64_t) * (size_t)rounds_cap);
      if (!np || !nc) {
        rc = fail(RPO_ENOMEM, "out of memory");
        goto done;
      }
      all_prop = np;
      all_cnt = nc;
    }
    memcpy(all_prop + round * b, proposed, sizeof(int64_t) * (size_t)b);
    all_cnt[round] = m;
  }
  /* finalize (rpcholesky.hpp:395-399, 140-145, 256-262) */
  res->n = n;
  res->rank = kcur;
  res->block_size = b;
  res->n_rounds = round;
  res->factor = f;
  f = NULL;
  res->pivots = pivots;
  pivots = NULL;
  res->chol = (double*)calloc((size_t)(kcur * kcur > 0 ? kcur * kcur : 1), sizeof(double));
  if (!res->chol) {
    rc = fail(RPO_ENOMEM, "out of memory");
    goto done;
  }
  for (int64_t j = 0; j < kcur; ++j)
    for (int64_t i = j; i < kcur; ++i) res->chol[j * kcur + i] = res->factor[j * n + res->pivots[i]];
  res->residual_diag = u;
  u = NULL;
  res->proposed = all_prop;
  all_prop = NULL;
  res->accepted_count = all_cnt;
  all_cnt = NULL;
  if (cfg->mode == RPO_MODE_UNTIL_RANK && kcur > cfg->target_rank) res->surplus = kcur - cfg->target_rank;
  res->captured_sq = captured_sq;
done:
  free(u);
  free(cumsum);
  free(f);
  free(pivots);
  free(proposed);
  free(h);
  free(fr);
  free(acc_ids);
  free(acc_pos);
  free(lsel);
  free(all_prop);
  free(all_cnt);
  if (rc) rpo_result_free(res);
  return rc;
}

int rpo_accelerated_rpcholesky(const rpo_oracle* o, const rpo_run_config* cfg, rpo_result* res) {
  return rpo_accelerated_rpcholesky_bounded(o, cfg, -1, res);
}

/* ---- block_rpcholesky rpcholesky.hpp:268-333 / simple_rpcholesky 206-246 ---- */
/* Cholesky of an m x m column-major block (the LLT the reference delegates to Eigen;
 * restated as the left-looking dot-product form, which is what oracle/eigen_shim's LLT
 * computes, so the restatement and the reference-through-shim agree bitwise).
 * Returns 0 on success, -1 on a non-positive pivot. */
static int llt_lower(const double* a, int64_t m, double* l) {
  memset(l, 0, sizeof(double) * (size_t)(m * m));
  for (int64_t j = 0; j < m; ++j) {
    double s = a[j * m + j];
    for (int64_t k = 0; k < j; ++k) s -= l[k * m + j] * l[k * m + j];
    if (!(s > 0.0)) return -1;
    const double dj = sqrt(s);
    l[j * m + j] = dj;
    for (int64_t i = j + 1; i < m; ++i) {
      double t = a[j * m + i];
      for (int64_t k = 0; k < j; ++k) t -= l[k * m + i] * l[k * m + j];
      l[j * m + i] = t / dj;
    }
  }
  return 0;
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}

/* algo 1: block (cfg as given); algo 2: simple (cfg = UntilRank(k, 1, seed)). */
static int rpo_block_or_simple(const rpo_oracle* o, const rpo_run_config* cfg, int algo,
                               rpo_result* res) {
  memset(res, 0, sizeof *res);
  const int64_t n = o->n;
  const int64_t b = cfg->block_size;
  const int nt = o->n_threads;
  const char* who = algo == 2 ? "simple_rpcholesky" : "block_rpcholesky";
  if (algo == 2 && (cfg->target_rank < 1 || cfg->target_rank > n))
    return fail(RPO_EINVAL, "simple_rpcholesky: need 1 <= k <= N");
  if (b < 1) return fail(RPO_EINVAL, "%s: block size must be >= 1", who);
  if (cfg->mode == RPO_MODE_FIXED_ROUNDS && cfg->rounds < 1)
    return fail(RPO_EINVAL, "RunConfig: t, b must be >= 1");
  if (cfg->mode == RPO_MODE_UNTIL_RANK && cfg->target_rank < 1)
    return fail(RPO_EINVAL, "RunConfig: k, b must be >= 1");
  double* dg = (double*)malloc(sizeof(double) * (size_t)n);
  double* cumsum = (double*)malloc(sizeof(double) * (size_t)n);
  if (!dg || !cumsum) {
    free(dg);
    free(cumsum);
    return fail(RPO_ENOMEM, "out of memory");
  }
  diag_of(o, dg);
  double trace_a = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (dg[i] < 0.0) dg[i] = 0.0;
    trace_a += dg[i];
  }
  if (!(trace_a > 0.0)) {
    free(dg);
    free(cumsum);
    return fail(RPO_EINVAL, "%s: trace must be > 0", who);
  }
  int64_t cap = algo == 2 ? cfg->target_rank
                          : (cfg->mode == RPO_MODE_FIXED_ROUNDS ? cfg->rounds * b : cfg->target_rank + b);
  if (cap > n) cap = n;
  double* f = (double*)malloc(sizeof(double) * (size_t)n * (size_t)cap);
  int64_t* pivots = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int64_t* proposed = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  double* fr = (double*)malloc(sizeof(double) * (size_t)(b * cap));
  double* blk = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* lsel = (double*)malloc(sizeof(double) * (size_t)(b * b));
  int64_t rounds_cap = 16;
  int64_t* all_prop = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rounds_cap * b));
  int64_t* all_cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)rounds_cap);
  int64_t* all_kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int rc = RPO_OK;
  if (!f || !pivots || !proposed || !kept || !fr || !blk || !lsel || !all_prop || !all_cnt ||
      !all_kept) {
    rc = fail(RPO_ENOMEM, "out of memory");
    goto done;
  }
  int64_t kcur = 0;
  double captured_sq = 0.0;
  uint64_t draw = 0;
  int64_t round;
  for (round = 0; !run_finished(cfg, round, kcur); ++round) {
    double usum = 0.0;
    for (int64_t i = 0; i < n; ++i) usum += dg[i];
    if (!(usum > 0.0)) {
      res->rank_exhausted = 1;
      break;
    }
    if (algo == 1 && cfg->stop_tol > 0.0 && (trace_a - captured_sq) <= cfg->stop_tol * trace_a) break;
    rpo_cumulative_sums(dg, n, cumsum);
    for (int64_t j = 0; j < b; ++j) {
      rc = rpo_sample_discrete(cumsum, n, rpo_u01(rpo_splitmix64_draw(cfg->seed, draw++)),
                               &proposed[j]);
      if (rc) goto done;
    }
    /* kept = unique_sorted(proposed) */
    memcpy(kept, proposed, sizeof(int64_t) * (size_t)b);
    qsort(kept, (size_t)b, sizeof(int64_t), cmp_i64);
    int64_t m = 0;
    for (int64_t j = 0; j < b; ++j)
      if (j == 0 || kept[j] != kept[m - 1]) kept[m++] = kept[j];
    if (kcur + m > cap) {
      rc = fail(RPO_ENUMERIC, "%s: factor capacity exceeded", who);
      goto done;
    }
    double* g = f + kcur * n;
    oracle_columns(o, kept, m, g);
    if (kcur > 0) {
      for (int64_t k = 0; k < kcur; ++k)
        for (int64_t i = 0; i < m; ++i) fr[k * m + i] = f[k * n + kept[i]];
      residual_gemm(f, n, kcur, fr, m, g, nt);
    }
    if (algo == 2) {
      /* simple: g / sqrt(g[s]); !(g[s] > 0) -> rank exhausted (229-236) */
      const double gs = g[kept[0]];
      if (!(gs > 0.0)) {
        res->rank_exhausted = 1;
        break;
      }
      const double root = sqrt(gs);
      for (int64_t i = 0; i < n; ++i) g[i] = g[i] / root;
    } else {
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i) blk[j * m + i] = g[j * n + kept[i]];
      if (llt_lower(blk, m, lsel) != 0) {
        const double shift = 64.0 * 2.220446049250313e-16 * trace_a / (double)n;
        for (int64_t i = 0; i < m; ++i) blk[i * m + i] += shift;
        if (llt_lower(blk, m, lsel) != 0) {
          rc = fail(RPO_ENUMERIC, "block_rpcholesky: Cholesky failed after diagonal shift");
          goto done;
        }
      }
      right_solve_lt(lsel, m, g, n, nt);
    }
    for (int64_t i = 0; i < n; ++i) {
      double s2 = 0.0;
      for (int64_t j = 0; j < m; ++j) s2 += g[j * n + i] * g[j * n + i];
      dg[i] -= s2;
    }
    for (int64_t i = 0; i < n; ++i)
      if (dg[i] < 0.0) dg[i] = 0.0;
    double gs2 = 0.0;
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < n; ++i) gs2 += g[j * n + i] * g[j * n + i];
    captured_sq += gs2;
    for (int64_t j = 0; j < m; ++j) pivots[kcur + j] = kept[j];
    kcur += m;
    if (round >= rounds_cap) {
      rounds_cap *= 2;
      int64_t* np = (int64_t*)realloc(all_prop, sizeof(int64_t) * (size_t)(rounds_cap * b));
      int64_t* nc = (int64_t*)realloc(all_cnt, sizeof(int64_t) * (size_t)rounds_cap);
      if (!np || !nc) {
        rc = fail(RPO_ENOMEM, "out of memory");
        goto done;
      }
      all_prop = np;
      all_cnt = nc;
    }
    memcpy(all_prop + round * b, proposed, sizeof(int64_t) * (size_t)b);
    all_cnt[round] = m;
  }
  res->n = n;
  res->rank = kcur;
  res->block_size = b;
  res->n_rounds = round;
  res->factor = f;
  f = NULL;
  res->pivots = pivots;
  pivots = NULL;
  res->chol = (double*)calloc((size_t)(kcur * kcur > 0 ? kcur * kcur : 1), sizeof(double));
  if (!res->chol) {
    rc = fail(RPO_ENOMEM, "out of memory");
    goto done;
  }
  for (int64_t j = 0; j < kcur; ++j)
    for (int64_t i = j; i < kcur; ++i) res->chol[j * kcur + i] = res->factor[j * n + res->pivots[i]];
  res->residual_diag = dg;
  dg = NULL;
  res->proposed = all_prop;
  all_prop = NULL;
  res->accepted_count = all_cnt;
  all_cnt = NULL;
  if (algo == 1 && cfg->mode == RPO_MODE_UNTIL_RANK && kcur > cfg->target_rank)
    res->surplus = kcur - cfg->target_rank;
  res->captured_sq = captured_sq;
done:
  free(dg);
  free(cumsum);
  free(f);
  free(pivots);
  free(proposed);
  free(kept);
  free(fr);
  free(blk);
  free(lsel);
  free(all_prop);
  free(all_cnt);
  free(all_kept);
  if (rc) rpo_result_free(res);
  return rc;
}

int rpo_block_rpcholesky(const rpo_oracle* o, const rpo_run_config* cfg, rpo_result* res) {
  return rpo_block_or_simple(o, cfg, 1, res);
}

int rpo_simple_rpcholesky(const rpo_oracle* o, int64_t k, uint64_t seed, rpo_result* res) {
  rpo_run_config c;
  memset(&c, 0, sizeof c);
  c.block_size = 1;
  c.mode = RPO_MODE_UNTIL_RANK;
  c.target_rank = k;
  c.seed = seed;
  return rpo_block_or_simple(o, &c, 2, res);
}

/* ---- rpcholesky.hpp:408-485  accelerated_rpcholesky_lowmem ---------- */
/* Forward substitution L y = w in place for nc columns (L: k x k column-major lower,
 * w: k x nc column-major with leading dimension ldw) — triangularView<Lower>::solveInPlace. */
static void lower_solve_inplace(const double* l, int64_t k, double* w, int64_t ldw, int64_t nc) {
  for (int64_t c = 0; c < nc; ++c) {
    double* y = w + c * ldw;
    for (int64_t i = 0; i < k; ++i) {
      double s = y[i];
      for (int64_t j = 0; j < i; ++j) s -= l[j * k + i] * y[j];
      y[i] = s / l[i * k + i];
    }
  }
}

int rpo_accelerated_rpcholesky_lowmem(const rpo_oracle* o, const rpo_run_config* cfg,
                                      rpo_result* res) {
  memset(res, 0, sizeof *res);
  const int64_t n = o->n;
  const int64_t b = cfg->block_size;
  const int nt = o->n_threads;
  if (b < 1) return fail(RPO_EINVAL, "accelerated_rpcholesky_lowmem: block size must be >= 1");
  if (cfg->mode == RPO_MODE_FIXED_ROUNDS && cfg->rounds < 1)
    return fail(RPO_EINVAL, "RunConfig: t, b must be >= 1");
  if (cfg->mode == RPO_MODE_UNTIL_RANK && cfg->target_rank < 1)
    return fail(RPO_EINVAL, "RunConfig: k, b must be >= 1");
  double* u = (double*)malloc(sizeof(double) * (size_t)n);
  double* cumsum = (double*)malloc(sizeof(double) * (size_t)n);
  if (!u || !cumsum) {
    free(u);
    free(cumsum);
    return fail(RPO_ENOMEM, "out of memory");
  }
  diag_of(o, u);
  double trace_a = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (u[i] < 0.0) u[i] = 0.0;
    trace_a += u[i];
  }
  if (!(trace_a > 0.0)) {
    free(u);
    free(cumsum);
    return fail(RPO_EINVAL, "accelerated_rpcholesky_lowmem: trace must be > 0");
  }
  int64_t cap = cfg->mode == RPO_MODE_FIXED_ROUNDS ? cfg->rounds * b : cfg->target_rank + b;
  if (cap > n) cap = n;
  if (cap < 1) cap = 1;
  const int64_t nchunks = (n + b - 1) / b;
  double* l = (double*)calloc((size_t)(cap * cap), sizeof(double)); /* k x k, ld = k (repacked) */
  double* lnext = (double*)calloc((size_t)(cap * cap), sizeof(double));
  int64_t* pivots = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int64_t* s_all = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int64_t* proposed = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  double* h = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* w_prop = (double*)malloc(sizeof(double) * (size_t)(cap * b));
  double* w_acc = (double*)malloc(sizeof(double) * (size_t)(cap * b));
  int64_t* acc_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  int64_t* acc_pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
  double* lsel = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* chunk_g2 = (double*)malloc(sizeof(double) * (size_t)nchunks);
  int64_t rounds_cap = 16;
  int64_t* all_prop = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rounds_cap * b));
  int64_t* all_cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)rounds_cap);
  int rc = RPO_OK;
  if (!l || !lnext || !pivots || !s_all || !proposed || !h || !w_prop || !w_acc || !acc_ids ||
      !acc_pos || !lsel || !chunk_g2 || !all_prop || !all_cnt) {
    rc = fail(RPO_ENOMEM, "out of memory");
    goto done;
  }
  int64_t kold = 0;
  double captured_sq = 0.0;
  uint64_t draw = 0;
  int64_t round;
  for (round = 0; !run_finished(cfg, round, kold); ++round) {
    double usum = 0.0;
    for (int64_t i = 0; i < n; ++i) usum += u[i];
    if (!(usum > 0.0)) { /* 423-426 */
      res->rank_exhausted = 1;
      break;
    }
    if (cfg->stop_tol > 0.0 && (trace_a - captured_sq) <= cfg->stop_tol * trace_a) break;
    rpo_cumulative_sums(u, n, cumsum);
    for (int64_t j = 0; j < b; ++j) {
      rc = rpo_sample_discrete(cumsum, n, rpo_u01(rpo_splitmix64_draw(cfg->seed, draw++)),
                               &proposed[j]);
      if (rc) goto done;
    }
    /* h = A(S', S') - W_prop^T W_prop, W_prop = L^{-1} A(S, S')  (438-445) */
    if ((rc = rpo_submatrix(o, proposed, b, proposed, b, h))) goto done;
    if (kold > 0) {
      if ((rc = rpo_submatrix(o, pivots, kold, proposed, b, w_prop))) goto done;
      lower_solve_inplace(l, kold, w_prop, kold, b);
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < b; ++i) {
          double s2 = 0.0;
          for (int64_t t = 0; t < kold; ++t) s2 += w_prop[i * kold + t] * w_prop[j * kold + t];
          h[j * b + i] -= s2;
        }
    }
    int64_t m = 0;
    if ((rc = rpo_rejection_sweep(h, b, proposed, cfg->seed, draw, acc_ids, acc_pos, &m, lsel)))
      goto done;
    draw += (uint64_t)b;
    if (m > 0) {
      if (kold + m > cap) {
        rc = fail(RPO_ENUMERIC, "accelerated_rpcholesky_lowmem: pivot capacity exceeded");
        goto done;
      }
      /* W_acc = W_prop(:, positions)  (449-455) */
      for (int64_t j = 0; j < m; ++j)
        for (int64_t t = 0; t < kold; ++t) w_acc[j * kold + t] = w_prop[acc_pos[j] * kold + t];
      const int64_t kn = kold + m;
      for (int64_t t = 0; t < kold; ++t) s_all[t] = pivots[t];
      for (int64_t j = 0; j < m; ++j) s_all[kold + j] = acc_ids[j];
      /* diagonal update in row chunks of b (457-468) */
#pragma omp parallel num_threads(nt)
      {
        double* a_chunk = (double*)malloc(sizeof(double) * (size_t)(b * kn));
        double* y = (double*)malloc(sizeof(double) * (size_t)(kold * b + 1));
        double* g = (double*)malloc(sizeof(double) * (size_t)(b * m));
        int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)b);
#pragma omp for schedule(static)
        for (int64_t ch = 0; ch < nchunks; ++ch) {
          const int64_t r0 = ch * b;
          const int64_t ht = (r0 + b <= n) ? b : n - r0;
          for (int64_t a = 0; a < ht; ++a) rows[a] = r0 + a;
          rpo_submatrix(o, rows, ht, s_all, kn, a_chunk); /* ht x kn, ld = ht */
          for (int64_t j = 0; j < m; ++j)
            for (int64_t a = 0; a < ht; ++a) g[j * ht + a] = a_chunk[(kold + j) * ht + a];
          if (kold > 0) {
            /* y = A(S_old, R) solved against L; g -= y^T W_acc */
            for (int64_t a = 0; a < ht; ++a)
              for (int64_t t = 0; t < kold; ++t) y[a * kold + t] = a_chunk[t * ht + a];
            lower_solve_inplace(l, kold, y, kold, ht);
            for (int64_t j = 0; j < m; ++j)
              for (int64_t a = 0; a < ht; ++a) {
                double s2 = 0.0;
                for (int64_t t = 0; t < kold; ++t) s2 += y[a * kold + t] * w_acc[j * kold + t];
                g[j * ht + a] -= s2;
              }
          }
          right_solve_lt(lsel, m, g, ht, 1);
          double gs = 0.0;
          for (int64_t a = 0; a < ht; ++a) {
            double s2 = 0.0;
            for (int64_t j = 0; j < m; ++j) s2 += g[j * ht + a] * g[j * ht + a];
            u[r0 + a] -= s2;
          }
          for (int64_t j = 0; j < m; ++j)
            for (int64_t a = 0; a < ht; ++a) gs += g[j * ht + a] * g[j * ht + a];
          chunk_g2[ch] = gs;
        }
        free(a_chunk);
        free(y);
        free(g);
        free(rows);
      }
      for (int64_t ch = 0; ch < nchunks; ++ch) captured_sq += chunk_g2[ch];
      /* l_next = [[l, 0], [W_acc^T, L_sel]]  (470-475) */
      memset(lnext, 0, sizeof(double) * (size_t)(kn * kn));
      for (int64_t c = 0; c < kold; ++c)
        for (int64_t r = 0; r < kold; ++r) lnext[c * kn + r] = l[c * kold + r];
      for (int64_t c = 0; c < kold; ++c)
        for (int64_t j = 0; j < m; ++j) lnext[c * kn + kold + j] = w_acc[j * kold + c];
      for (int64_t c = 0; c < m; ++c)
        for (int64_t j = 0; j < m; ++j) lnext[(kold + c) * kn + kold + j] = lsel[c * m + j];
      double* tmp = l;
      l = lnext;
      lnext = tmp;
      for (int64_t j = 0; j < m; ++j) pivots[kold + j] = acc_ids[j];
      kold = kn;
    }
    for (int64_t i = 0; i < n; ++i)
      if (u[i] < 0.0) u[i] = 0.0; /* 478 */
    if (round >= rounds_cap) {
      rounds_cap *= 2;
      int64_t* np = (int64_t*)realloc(all_prop, sizeof(int64_t) * (size_t)(rounds_cap * b));
      int64_t* nc = (int64_t*)realloc(all_cnt, sizeof(int64_t) * (size_t)rounds_cap);
      if (!np || !nc) {
        rc = fail(RPO_ENOMEM, "out of memory");
        goto done;
      }
      all_prop = np;
      all_cnt = nc;
    }
    memcpy(all_prop + round * b, proposed, sizeof(int64_t) * (size_t)b);
    all_cnt[round] = m;
  }
  res->n = n;
  res->rank = kold;
  res->block_size = b;
  res->n_rounds = round;
  res->factor = NULL; /* LowMemResult has no factor (114-119) */
  res->pivots = pivots;
  pivots = NULL;
  res->chol = l;
  l = NULL;
  res->residual_diag = u;
  u = NULL;
  res->proposed = all_prop;
  all_prop = NULL;
  res->accepted_count = all_cnt;
  all_cnt = NULL;
  if (cfg->mode == RPO_MODE_UNTIL_RANK && kold > cfg->target_rank) res->surplus = kold - cfg->target_rank;
  res->captured_sq = captured_sq;
done:
  free(u);
  free(cumsum);
  free(l);
  free(lnext);
  free(pivots);
  free(s_all);
  free(proposed);
  free(h);
  free(w_prop);
  free(w_acc);
  free(acc_ids);
  free(acc_pos);
  free(lsel);
  free(chunk_g2);
  free(all_prop);
  free(all_cnt);
  if (rc) rpo_result_free(res);
  return rc;
}

void rpo_result_free(rpo_result* res) {
  free(res->factor);
  free(res->pivots);
  free(res->chol);
  free(res->residual_diag);
  free(res->proposed);
  free(res->accepted_count);
  memset(res, 0, sizeof *res);
}

/* ---- rpcholesky.hpp:577-583  relative_trace_error -------------------- */
double rpo_relative_trace_error(const rpo_oracle* o, const double* factor, int64_t n, int64_t k) {
  double* dg = (double*)malloc(sizeof(double) * (size_t)n);
  diag_of(o, dg);
  double tr = 0.0;
  for (int64_t i = 0; i < n; ++i) tr += dg[i];
  free(dg);
  double fs = 0.0;
  for (int64_t i = 0; i < n * k; ++i) fs += factor[i] * factor[i];
  double err = (tr - fs) / tr;
  if (err < 0.0) err = 0.0;
  if (err > 1.0) err = 1.0;
  return err;
}
