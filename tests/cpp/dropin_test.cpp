// Drop-in check: the reference's own types and CPU path against rpchol::b200.
//
// Built by `make -C oracle dropin` (needs the reference headers, compiled against the
// Eigen-API shim) into oracle/_ref/dropin_test; run on a B200 by tests/test_dropin.py.
// A reference user swaps rpchol::accelerated_rpcholesky for
// rpchol::b200::accelerated_rpcholesky with the same KernelOracle and RunConfig (and
// accelerated_rpcholesky_lowmem for rpchol::b200::accelerated_rpcholesky_lowmem).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "rpchol_b200.hpp"

using namespace rpchol;

static int fails = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
      ++fails;                                                      \
    }                                                               \
  } while (0)

static double rel(const Eigen::MatrixXd& a, const Eigen::MatrixXd& b) {
  const double nb = b.norm();
  Eigen::MatrixXd d = a - b;
  return nb > 0 ? d.norm() / nb : d.norm();
}

static void compare(const char* name, const PsdOracle& oracle, const RunConfig& cfg) {
  const CholeskyResult ref = rpchol::accelerated_rpcholesky(oracle, cfg);
  const CholeskyResult gpu = rpchol::b200::accelerated_rpcholesky(oracle, cfg);
  EXPECT(ref.approx.pivots == gpu.approx.pivots);
  EXPECT(ref.trace.rounds.size() == gpu.trace.rounds.size());
  for (size_t r = 0; r < std::min(ref.trace.rounds.size(), gpu.trace.rounds.size()); ++r) {
    EXPECT(ref.trace.rounds[r].proposed == gpu.trace.rounds[r].proposed);
    EXPECT(ref.trace.rounds[r].accepted == gpu.trace.rounds[r].accepted);
  }
  EXPECT(ref.trace.rank_exhausted == gpu.trace.rank_exhausted);
  EXPECT(ref.trace.surplus == gpu.trace.surplus);
  const double ef = rel(gpu.approx.factor, ref.approx.factor);
  const double ec = rel(gpu.approx.chol_factor, ref.approx.chol_factor);
  const double eu = rel(gpu.residual_diag, ref.residual_diag);
  EXPECT(ef <= 1e-10);
  EXPECT(ec <= 1e-10);
  EXPECT(eu <= 1e-10);
  const double tr = std::abs(relative_trace_error(oracle, gpu.approx) -
                             relative_trace_error(oracle, ref.approx));
  EXPECT(tr <= 1e-8);
  std::printf("%s: rank %ld rounds %zu  |dF|/|F| %.2e  |dL|/|L| %.2e  |du|/|u| %.2e  dtrace %.2e\n",
              name, (long)gpu.approx.rank(), gpu.trace.rounds.size(), ef, ec, eu, tr);
}

static void compare_lowmem(const char* name, const PsdOracle& oracle, const RunConfig& cfg) {
  const LowMemResult ref = rpchol::accelerated_rpcholesky_lowmem(oracle, cfg);
  const LowMemResult gpu = rpchol::b200::accelerated_rpcholesky_lowmem(oracle, cfg);
  EXPECT(ref.pivots == gpu.pivots);
  EXPECT(ref.trace.rounds.size() == gpu.trace.rounds.size());
  for (size_t r = 0; r < std::min(ref.trace.rounds.size(), gpu.trace.rounds.size()); ++r) {
    EXPECT(ref.trace.rounds[r].proposed == gpu.trace.rounds[r].proposed);
    EXPECT(ref.trace.rounds[r].accepted == gpu.trace.rounds[r].accepted);
  }
  EXPECT(ref.trace.rank_exhausted == gpu.trace.rank_exhausted);
  EXPECT(ref.trace.surplus == gpu.trace.surplus);
  const double ec = rel(gpu.chol_factor, ref.chol_factor);
  const double eu = (gpu.residual_diag - ref.residual_diag).cwiseAbs().maxCoeff();
  EXPECT(ec <= 1e-10);
  EXPECT(eu <= 1e-8);
  std::printf("%s (lowmem): rank %zu rounds %zu  |dL|/|L| %.2e  max|du| %.2e\n", name,
              gpu.pivots.size(), gpu.trace.rounds.size(), ec, eu);
}

int main() {
  SplitMix64 rng(0);
  const Eigen::Index n = 6000, d = 10;
  Eigen::MatrixXd x(n, d);
  for (Eigen::Index i = 0; i < n; ++i)
    for (Eigen::Index j = 0; j < d; ++j) x(i, j) = sample_standard_normal(rng);
  KernelOracle gauss(DataMatrix(x), KernelSpec(KernelKind::Gaussian, std::sqrt(10.0)));
  compare("gaussian-gram until_rank(200, 40)", gauss, RunConfig::until_rank(200, 40, 0));
  compare("gaussian-gram fixed_rounds(5, 17)", gauss, RunConfig::fixed_rounds(5, 17, 3));
  KernelOracle l1(DataMatrix(x), KernelSpec(KernelKind::L1Laplace, 5.0));
  compare("l1 until_rank(150, 60)", l1, RunConfig::until_rank(150, 60, 1));
  KernelOracle direct(DataMatrix(x), KernelSpec(KernelKind::Gaussian, 2.0), DistanceMode::Direct);
  compare("gaussian-direct until_rank(100, 25)", direct, RunConfig::until_rank(100, 25, 2));
  KernelOracle m32(DataMatrix(x), KernelSpec(KernelKind::Matern32, 2.0));
  compare("matern32-gram until_rank(150, 40)", m32, RunConfig::until_rank(150, 40, 4));
  KernelOracle m52(DataMatrix(x), KernelSpec(KernelKind::Matern52, 2.0), DistanceMode::Direct);
  compare("matern52-direct fixed_rounds(4, 30)", m52, RunConfig::fixed_rounds(4, 30, 5));
  compare_lowmem("gaussian-gram until_rank(200, 40)", gauss, RunConfig::until_rank(200, 40, 0));
  compare_lowmem("l1 fixed_rounds(4, 60)", l1, RunConfig::fixed_rounds(4, 60, 1));

  // error behaviour mirrors the reference
  try {
    RunConfig bad = RunConfig::until_rank(10, 4, 0);
    bad.block_size = 0;
    rpchol::b200::accelerated_rpcholesky(gauss, bad);
    EXPECT(false);
  } catch (const std::invalid_argument& e) {
    EXPECT(std::string(e.what()) == "accelerated_rpcholesky: block size must be >= 1");
  }
  try {
    DenseOracle dense(Eigen::MatrixXd::Identity(4, 4));
    rpchol::b200::accelerated_rpcholesky(dense, RunConfig::until_rank(2, 1, 0));
    EXPECT(false);
  } catch (const std::invalid_argument&) {
  }
  std::printf(fails ? "DROPIN FAILED (%d)\n" : "DROPIN OK\n", fails);
  return fails ? 1 : 0;
}
