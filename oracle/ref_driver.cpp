// ref_driver.cpp — C entry points around the REFERENCE's own headers
// (/root/reference/proj/include/rpchol, compiled where they lie against the
// Eigen-API shim in oracle/eigen_shim).  TEST INFRASTRUCTURE ONLY: it produces
// oracle/_ref/libref_rpchol.so, used by tests/ to pin the C restatement
// (oracle/rpc_oracle.c) against the reference's actual control flow and
// arithmetic, and by bench.py's --impl reference arm.  No reference source is
// copied into this repository.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpchol/io.hpp"
#include "rpchol/krr.hpp"
#include "rpchol/rpcholesky.hpp"

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  return 3;
}

// Same layout as rpo_result (oracle/rpc_oracle.h) so the Python binding is shared.
struct Res {
  int64_t n, rank;
  double* factor;
  int64_t* pivots;
  double* chol;
  double* residual_diag;
  int64_t n_rounds, block_size;
  int64_t* proposed;
  int64_t* accepted_count;
  int rank_exhausted;
  int64_t surplus;
  double captured_sq;
};

template <class T>
T* dup(const T* src, size_t n) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (n ? n : 1)));
  if (n) std::memcpy(p, src, sizeof(T) * n);
  return p;
}

rpchol::RunConfig make_cfg(int64_t b, int mode, int64_t rounds, int64_t k, uint64_t seed,
                           double stop_tol) {
  rpchol::RunConfig cfg = mode == 0 ? rpchol::RunConfig::fixed_rounds(rounds, b, seed)
                                    : rpchol::RunConfig::until_rank(k, b, seed);
  cfg.stop_tol = stop_tol;
  return cfg;
}

void fill(const rpchol::CholeskyResult& r, Res* out, int64_t b) {
  const auto& f = r.approx.factor;
  out->n = f.rows();
  out->rank = f.cols();
  out->factor = dup(f.data(), (size_t)(f.rows() * f.cols()));
  std::vector<int64_t> piv(r.approx.pivots.begin(), r.approx.pivots.end());
  out->pivots = dup(piv.data(), piv.size());
  out->chol = dup(r.approx.chol_factor.data(),
                  (size_t)(r.approx.chol_factor.rows() * r.approx.chol_factor.cols()));
  out->residual_diag = dup(r.residual_diag.data(), (size_t)r.residual_diag.size());
  out->n_rounds = (int64_t)r.trace.rounds.size();
  out->block_size = b;
  std::vector<int64_t> prop, cnt;
  for (const auto& rr : r.trace.rounds) {
    prop.insert(prop.end(), rr.proposed.begin(), rr.proposed.end());
    cnt.push_back((int64_t)rr.accepted.size());
  }
  out->proposed = dup(prop.data(), prop.size());
  out->accepted_count = dup(cnt.data(), cnt.size());
  out->rank_exhausted = r.trace.rank_exhausted ? 1 : 0;
  out->surplus = r.trace.surplus;
  out->captured_sq = 0.0;
}

rpchol::KernelKind kind_of(int kind) {
  switch (kind) {
    case 0: return rpchol::KernelKind::Gaussian;
    case 1: return rpchol::KernelKind::L1Laplace;
    case 2: return rpchol::KernelKind::Matern32;
    default: return rpchol::KernelKind::Matern52;
  }
}

rpchol::KernelOracle make_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma,
                                 int dist) {
  Eigen::MatrixXd pts(n, d);
  std::memcpy(pts.data(), x, sizeof(double) * (size_t)(n * d));
  rpchol::KernelSpec spec(kind_of(kind), sigma);
  return rpchol::KernelOracle(rpchol::DataMatrix(std::move(pts)), spec,
                              dist == 1 ? rpchol::DistanceMode::GramTrick
                                        : rpchol::DistanceMode::Direct);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// x: n x d column-major.  dist: 0 direct, 1 gram.
int ref_accelerated_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                           int64_t b, int mode, int64_t rounds, int64_t k, uint64_t seed,
                           double stop_tol, Res* out) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    auto res = rpchol::accelerated_rpcholesky(oracle, make_cfg(b, mode, rounds, k, seed, stop_tol));
    fill(res, out, b);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

int ref_accelerated_dense(const double* a, int64_t n, int64_t b, int mode, int64_t rounds,
                          int64_t k, uint64_t seed, double stop_tol, Res* out) {
  try {
    Eigen::MatrixXd m(n, n);
    std::memcpy(m.data(), a, sizeof(double) * (size_t)(n * n));
    rpchol::DenseOracle oracle(std::move(m));
    auto res = rpchol::accelerated_rpcholesky(oracle, make_cfg(b, mode, rounds, k, seed, stop_tol));
    fill(res, out, b);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// block_rpcholesky (rpcholesky.hpp:268-333)
int ref_block_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                     int64_t b, int mode, int64_t rounds, int64_t k, uint64_t seed,
                     double stop_tol, Res* out) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    auto res = rpchol::block_rpcholesky(oracle, make_cfg(b, mode, rounds, k, seed, stop_tol));
    fill(res, out, b);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// simple_rpcholesky (rpcholesky.hpp:206-246)
int ref_simple_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                      int64_t k, uint64_t seed, Res* out) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    auto res = rpchol::simple_rpcholesky(oracle, k, seed);
    fill(res, out, 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485): factor = NULL, rank = |pivots|.
int ref_lowmem_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                      int64_t b, int mode, int64_t rounds, int64_t k, uint64_t seed,
                      double stop_tol, Res* out) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    auto r = rpchol::accelerated_rpcholesky_lowmem(oracle, make_cfg(b, mode, rounds, k, seed, stop_tol));
    std::memset(out, 0, sizeof *out);
    out->n = n;
    out->rank = (int64_t)r.pivots.size();
    std::vector<int64_t> piv(r.pivots.begin(), r.pivots.end());
    out->pivots = dup(piv.data(), piv.size());
    out->chol = dup(r.chol_factor.data(), (size_t)(r.chol_factor.rows() * r.chol_factor.cols()));
    out->residual_diag = dup(r.residual_diag.data(), (size_t)r.residual_diag.size());
    out->n_rounds = (int64_t)r.trace.rounds.size();
    out->block_size = b;
    std::vector<int64_t> prop, cnt;
    for (const auto& rr : r.trace.rounds) {
      prop.insert(prop.end(), rr.proposed.begin(), rr.proposed.end());
      cnt.push_back((int64_t)rr.accepted.size());
    }
    out->proposed = dup(prop.data(), prop.size());
    out->accepted_count = dup(cnt.data(), cnt.size());
    out->rank_exhausted = r.trace.rank_exhausted ? 1 : 0;
    out->surplus = r.trace.surplus;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

double ref_relative_trace_error_kernel(const double* x, int64_t n, int64_t d, int kind,
                                       double sigma, int dist, const double* factor, int64_t k) {
  auto oracle = make_kernel(x, n, d, kind, sigma, dist);
  rpchol::LowRankApprox approx;
  approx.factor.resize(n, k);
  std::memcpy(approx.factor.data(), factor, sizeof(double) * (size_t)(n * k));
  return rpchol::relative_trace_error(oracle, approx);
}

int ref_kernel_submatrix(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                         const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                         double* out) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    std::vector<Eigen::Index> r(rows, rows + nr), c(cols, cols + nc);
    Eigen::MatrixXd m = oracle.submatrix(r, c);
    std::memcpy(out, m.data(), sizeof(double) * (size_t)(nr * nc));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

int ref_sample_discrete(const double* w, int64_t n, uint64_t seed, uint64_t draw0, int64_t count,
                        int64_t* out) {
  try {
    Eigen::VectorXd wv(n);
    std::memcpy(wv.data(), w, sizeof(double) * (size_t)n);
    const Eigen::VectorXd cs = rpchol::cumulative_sums(wv);
    rpchol::SplitMix64 rng(seed);
    for (uint64_t t = 0; t < draw0; ++t) rng.next_u64();
    for (int64_t j = 0; j < count; ++j) out[j] = rpchol::sample_discrete(cs, rng);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

int ref_rejection_sweep(const double* h, int64_t b, const int64_t* proposals, uint64_t seed,
                        uint64_t draw0, int64_t* accepted, int64_t* positions, int64_t* m_out,
                        double* chol) {
  try {
    Eigen::MatrixXd hm(b, b);
    std::memcpy(hm.data(), h, sizeof(double) * (size_t)(b * b));
    std::vector<Eigen::Index> prop(proposals, proposals + b);
    rpchol::SplitMix64 rng(seed);
    for (uint64_t t = 0; t < draw0; ++t) rng.next_u64();
    auto sel = rpchol::rejection_sample_submatrix(std::move(hm), prop, rng);
    const int64_t m = (int64_t)sel.accepted.size();
    for (int64_t i = 0; i < m; ++i) {
      accepted[i] = sel.accepted[(size_t)i];
      positions[i] = sel.positions[(size_t)i];
    }
    std::memcpy(chol, sel.chol_factor.data(), sizeof(double) * (size_t)(m * m));
    *m_out = m;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// kernel_matvec (krr.hpp:143-162) with the oracle's DistanceMode.
int ref_kernel_matvec(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                      const double* v, int64_t row_block, double* out) {
  try {
    Eigen::MatrixXd pts(n, d);
    std::memcpy(pts.data(), x, sizeof(double) * (size_t)(n * d));
    rpchol::DataMatrix data(std::move(pts));
    rpchol::KernelSpec spec(kind_of(kind), sigma);
    Eigen::VectorXd vv(n);
    std::memcpy(vv.data(), v, sizeof(double) * (size_t)n);
    Eigen::VectorXd o = rpchol::kernel_matvec(
        data, spec, dist == 1 ? rpchol::DistanceMode::GramTrick : rpchol::DistanceMode::Direct, vv,
        row_block, 1);
    std::memcpy(out, o.data(), sizeof(double) * (size_t)n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// fit_krr (krr.hpp:177-224) + predict (227-250) on `query` (nq x d, col-major; may be null).
// rel / unreg / pivots need max_iters / max_iters / precond_rank entries.
int ref_fit_krr(const double* x, int64_t n, int64_t d, int kind, double sigma,
                const double* targets, double mu, int64_t precond_rank, int64_t b, uint64_t seed,
                double tol, int64_t max_iters, int64_t materialize_threshold, double* coef,
                double* mean, int64_t* iters, int* converged, double* rel, double* unreg,
                int64_t* pivots, int64_t* k_out, const double* query, int64_t nq, double* pred) {
  try {
    Eigen::MatrixXd pts(n, d);
    std::memcpy(pts.data(), x, sizeof(double) * (size_t)(n * d));
    rpchol::DataMatrix data(std::move(pts));
    rpchol::KernelSpec spec(kind_of(kind), sigma);
    Eigen::VectorXd t(n);
    std::memcpy(t.data(), targets, sizeof(double) * (size_t)n);
    rpchol::KrrOptions opts;
    opts.max_iters = max_iters;
    opts.materialize_threshold = materialize_threshold;
    auto fit = rpchol::fit_krr(data, t, spec, mu, precond_rank,
                               rpchol::RunConfig::until_rank(std::max<int64_t>(precond_rank, 1), b, seed),
                               tol, opts);
    std::memcpy(coef, fit.model.coefficients.data(), sizeof(double) * (size_t)n);
    *mean = fit.model.target_mean;
    *iters = fit.report.iterations;
    *converged = fit.report.converged ? 1 : 0;
    for (size_t i = 0; i < fit.report.relative_residuals.size(); ++i) {
      rel[i] = fit.report.relative_residuals[i];
      unreg[i] = fit.report.relative_residuals_unreg[i];
    }
    *k_out = (int64_t)fit.preconditioner.pivots.size();
    for (size_t i = 0; i < fit.preconditioner.pivots.size(); ++i) pivots[i] = fit.preconditioner.pivots[i];
    if (query && nq > 0) {
      Eigen::MatrixXd q(nq, d);
      std::memcpy(q.data(), query, sizeof(double) * (size_t)(nq * d));
      Eigen::VectorXd p = rpchol::predict(fit.model, rpchol::DataMatrix(std::move(q)));
      std::memcpy(pred, p.data(), sizeof(double) * (size_t)nq);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// read_rpcf (io.hpp:258-293) -> Res (factor, pivots, chol; chol empty -> rank x rank zeros)
int ref_read_rpcf(const char* path, Res* out) {
  try {
    rpchol::LowRankApprox a = rpchol::read_rpcf(path);
    std::memset(out, 0, sizeof *out);
    out->n = a.factor.rows();
    out->rank = a.factor.cols();
    out->factor = dup(a.factor.data(), (size_t)(a.factor.rows() * a.factor.cols()));
    std::vector<int64_t> piv(a.pivots.begin(), a.pivots.end());
    out->pivots = dup(piv.data(), piv.size());
    Eigen::MatrixXd c = a.chol_factor.rows() ? a.chol_factor
                                             : Eigen::MatrixXd::Zero(a.factor.cols(), a.factor.cols());
    out->chol = dup(c.data(), (size_t)(c.rows() * c.cols()));
    Eigen::VectorXd z = Eigen::VectorXd::Zero(out->n);
    out->residual_diag = dup(z.data(), (size_t)out->n);
    out->proposed = dup<int64_t>(nullptr, 0);
    out->accepted_count = dup<int64_t>(nullptr, 0);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

// write_rpcf (io.hpp:218-256) of a reference accelerated run -> the reference's own bytes
int ref_write_rpcf_kernel(const double* x, int64_t n, int64_t d, int kind, double sigma, int dist,
                          int64_t b, int64_t k, uint64_t seed, const char* path,
                          const char* trace_csv) {
  try {
    auto oracle = make_kernel(x, n, d, kind, sigma, dist);
    auto res = rpchol::accelerated_rpcholesky(oracle, rpchol::RunConfig::until_rank(k, b, seed));
    rpchol::write_rpcf(path, res.approx);
    if (trace_csv) rpchol::write_pivot_trace_csv(trace_csv, res.trace);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

void ref_result_free(Res* r) {
  std::free(r->factor);
  std::free(r->pivots);
  std::free(r->chol);
  std::free(r->residual_diag);
  std::free(r->proposed);
  std::free(r->accepted_count);
  std::memset(r, 0, sizeof *r);
}

}  // extern "C"
