// rpchol_b200.hpp — C++ drop-in for the reference's hot path on B200.
//
// A reference user replaces
//     rpchol::CholeskyResult res = rpchol::accelerated_rpcholesky(oracle, cfg);
// (/root/reference/proj/include/rpchol/rpcholesky.hpp:338-401) with
//     rpchol::CholeskyResult res = rpchol::b200::accelerated_rpcholesky(oracle, cfg);
// Same inputs (the reference's own KernelOracle / RunConfig types), same output type
// (CholeskyResult with factor, pivots, chol_factor, PivotTrace, residual_diag), same
// exception classes and messages.  Likewise accelerated_rpcholesky_lowmem
// (rpcholesky.hpp:408-485) -> rpchol::b200::accelerated_rpcholesky_lowmem (LowMemResult).  The computation runs in librpchol_b200.so through the
// C-ABI of rpchol_gpu.h.  Only KernelOracle inputs are accepted: any other PsdOracle
// throws std::invalid_argument (there is no CPU fallback).
//
// Requires the reference headers (and therefore Eigen) on the include path, exactly as
// the code it replaces does; link with -lrpchol_b200.
#ifndef RPCHOL_B200_HPP
#define RPCHOL_B200_HPP

#include <algorithm>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpchol/rpcholesky.hpp"
#include "rpchol_gpu.h"

namespace rpchol {
namespace b200 {

[[noreturn]] inline void throw_status(int code, const char* msg) {
  switch (code) {
    case RPC_EINVAL: throw std::invalid_argument(msg);
    case RPC_ERANGE: throw std::out_of_range(msg);
    case RPC_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

/// One B200 (or one rank of a multi-GPU job).  Not re-entrant; distinct
/// Devices on distinct GPUs may run concurrently.
class Device {
 public:
  explicit Device(int device = 0) {
    if (int rc = rpc_create(device, &ctx_)) throw_status(rc, rpc_last_error(nullptr));
  }
  Device(int device, const void* nccl_id128, int nranks, int rank) {
    if (int rc = rpc_create_nccl(device, nccl_id128, nranks, rank, &ctx_))
      throw_status(rc, rpc_last_error(nullptr));
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  ~Device() { rpc_destroy(ctx_); }
  rpc_ctx* get() const noexcept { return ctx_; }

 private:
  rpc_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
  static Device dev(0);
  return dev;
}

namespace detail {

using ResultPtr = std::unique_ptr<rpc_result, void (*)(rpc_result*)>;
using Entry = std::function<int(rpc_ctx*, const double*, int64_t, int64_t, int64_t, int,
                                rpc_kernel_spec, rpc_run_config, rpc_result**)>;

// Runs `entry` (standard or low-memory) on a KernelOracle; throws like the reference.
inline ResultPtr run(const PsdOracle& oracle, const RunConfig& cfg, Device& dev, const Entry& entry,
                     const char* who) {
  const auto* ko = dynamic_cast<const KernelOracle*>(&oracle);
  if (!ko) throw std::invalid_argument(std::string(who) + " (B200): only KernelOracle inputs are supported");
  const Eigen::MatrixXd& x = ko->data().points();  // N x d, column-major
  rpc_kernel_spec ks;
  switch (ko->kernel().kind) {
    case KernelKind::Gaussian: ks.kind = RPC_KERNEL_GAUSSIAN; break;
    case KernelKind::L1Laplace: ks.kind = RPC_KERNEL_L1LAPLACE; break;
    case KernelKind::Matern32: ks.kind = RPC_KERNEL_MATERN32; break;
    case KernelKind::Matern52: ks.kind = RPC_KERNEL_MATERN52; break;
    default:
      throw std::invalid_argument(std::string(who) + " (B200): unsupported kernel kind " +
                                  kernel_kind_name(ko->kernel().kind));
  }
  ks.sigma = ko->kernel().bandwidth;
  ks.distance_mode =
      ko->distance_mode() == DistanceMode::GramTrick ? RPC_DIST_GRAM : RPC_DIST_DIRECT;
  rpc_run_config rc;
  rc.block_size = cfg.block_size;
  rc.mode = cfg.mode == RunConfig::Mode::FixedRounds ? RPC_FIXED_ROUNDS : RPC_UNTIL_RANK;
  rc.rounds = cfg.rounds;
  rc.target_rank = cfg.target_rank;
  rc.seed = cfg.seed;
  rc.stop_tol = cfg.stop_tol;
  rc.flags = 0;
  rpc_result* raw = nullptr;
  if (int st = entry(dev.get(), x.data(), x.rows(), x.cols(), x.rows(), RPC_COL_MAJOR, ks, rc, &raw))
    throw_status(st, rpc_last_error(dev.get()));
  return ResultPtr(raw, rpc_result_free);
}

inline IndexList pivots_of(rpc_result* r) {
  const int64_t k = rpc_result_rank(r);
  std::vector<int64_t> buf(static_cast<std::size_t>(k));
  if (k > 0) rpc_result_pivots(r, buf.data());
  return IndexList(buf.begin(), buf.end());
}

inline Eigen::MatrixXd chol_of(rpc_result* r) {
  const Eigen::Index k = rpc_result_rank(r);
  Eigen::MatrixXd c(k, k);
  if (k > 0) rpc_result_chol_copy(r, c.data());
  return c;
}

inline Eigen::VectorXd residual_of(rpc_result* r) {
  Eigen::VectorXd u(rpc_result_n(r));
  rpc_result_residual_diag_copy(r, u.data());
  return u;
}

inline PivotTrace trace_of(rpc_result* r) {
  PivotTrace t;
  const int64_t b = rpc_result_block_size(r);
  std::vector<int64_t> prop(static_cast<std::size_t>(b)), acc(static_cast<std::size_t>(b));
  for (int64_t i = 0; i < rpc_result_num_rounds(r); ++i) {
    int64_t na = 0;
    rpc_result_round(r, i, prop.data(), acc.data(), &na);
    RoundRecord rec;
    rec.proposed.assign(prop.begin(), prop.end());
    rec.accepted.assign(acc.begin(), acc.begin() + na);
    t.rounds.push_back(std::move(rec));
  }
  t.rank_exhausted = rpc_result_rank_exhausted(r) != 0;
  t.surplus = rpc_result_surplus(r);
  return t;
}

}  // namespace detail

/// accelerated_rpcholesky (rpcholesky.hpp:338-401) for kernel oracles, on B200.
inline CholeskyResult accelerated_rpcholesky(const PsdOracle& oracle, const RunConfig& cfg,
                                             Device& dev = default_device()) {
  // the factor streams into res.approx.factor while the rounds run
  // (rpc_accelerated_rpcholesky_into), sized like the reference's (rpcholesky.hpp:348-351)
  const Eigen::Index n = oracle.dimension();
  const Eigen::Index cap = std::min<Eigen::Index>(
      n, cfg.mode == RunConfig::Mode::FixedRounds ? cfg.rounds * cfg.block_size
                                                  : cfg.target_rank + cfg.block_size);
  CholeskyResult res;
  res.approx.factor.resize(n, std::max<Eigen::Index>(cap, 1));
  double* fbuf = res.approx.factor.data();
  const Eigen::Index fcols = res.approx.factor.cols();
  auto r = detail::run(
      oracle, cfg, dev,
      [fbuf, n, fcols](rpc_ctx* c, const double* x, int64_t nn, int64_t d, int64_t ldx, int lay,
                       rpc_kernel_spec ks, rpc_run_config rc, rpc_result** out) {
        return rpc_accelerated_rpcholesky_into(c, x, nn, d, ldx, lay, ks, rc, fbuf, n, fcols, out);
      },
      "accelerated_rpcholesky");
  const Eigen::Index k = rpc_result_rank(r.get());
  res.approx.factor.conservativeResize(n, k);
  res.approx.pivots = detail::pivots_of(r.get());
  res.approx.chol_factor = detail::chol_of(r.get());
  res.residual_diag = detail::residual_of(r.get());
  res.trace = detail::trace_of(r.get());
  return res;
}

/// accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485) for kernel oracles, on B200:
/// O(N + k^2) device state, the N x k factor is never formed.
inline LowMemResult accelerated_rpcholesky_lowmem(const PsdOracle& oracle, const RunConfig& cfg,
                                                  Device& dev = default_device()) {
  auto r = detail::run(oracle, cfg, dev, rpc_accelerated_rpcholesky_lowmem,
                       "accelerated_rpcholesky_lowmem");
  LowMemResult res;
  res.pivots = detail::pivots_of(r.get());
  res.chol_factor = detail::chol_of(r.get());
  res.residual_diag = detail::residual_of(r.get());
  res.trace = detail::trace_of(r.get());
  return res;
}

}  // namespace b200
}  // namespace rpchol

#endif  // RPCHOL_B200_HPP
