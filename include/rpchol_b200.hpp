// rpchol_b200.hpp — C++ drop-in for the reference's hot path on B200.
//
// A reference user replaces
//     rpchol::CholeskyResult res = rpchol::accelerated_rpcholesky(oracle, cfg);
// (/root/reference/proj/include/rpchol/rpcholesky.hpp:338-401) with
//     rpchol::CholeskyResult res = rpchol::b200::accelerated_rpcholesky(oracle, cfg);
// Same inputs (the reference's own KernelOracle / RunConfig types), same output type
// (CholeskyResult with factor, pivots, chol_factor, PivotTrace, residual_diag), same
// exception classes and messages.  The computation runs in librpchol_b200.so through the
// C-ABI of rpchol_gpu.h.  Only KernelOracle inputs are accepted: any other PsdOracle
// throws std::invalid_argument (there is no CPU fallback).
//
// Requires the reference headers (and therefore Eigen) on the include path, exactly as
// the code it replaces does; link with -lrpchol_b200.
#ifndef RPCHOL_B200_HPP
#define RPCHOL_B200_HPP

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

/// accelerated_rpcholesky (rpcholesky.hpp:338-401) for kernel oracles, on B200.
inline CholeskyResult accelerated_rpcholesky(const PsdOracle& oracle, const RunConfig& cfg,
                                             Device& dev = default_device()) {
  const auto* ko = dynamic_cast<const KernelOracle*>(&oracle);
  if (!ko) {
    throw std::invalid_argument(
        "accelerated_rpcholesky (B200): only KernelOracle inputs are supported");
  }
  const Eigen::MatrixXd& x = ko->data().points();  // N x d, column-major
  rpc_kernel_spec ks;
  switch (ko->kernel().kind) {
    case KernelKind::Gaussian: ks.kind = RPC_KERNEL_GAUSSIAN; break;
    case KernelKind::L1Laplace: ks.kind = RPC_KERNEL_L1LAPLACE; break;
    default:
      throw std::invalid_argument("accelerated_rpcholesky (B200): unsupported kernel kind " +
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
  if (int st = rpc_accelerated_rpcholesky(dev.get(), x.data(), x.rows(), x.cols(), x.rows(),
                                          RPC_COL_MAJOR, ks, rc, &raw))
    throw_status(st, rpc_last_error(dev.get()));
  std::unique_ptr<rpc_result, void (*)(rpc_result*)> r(raw, rpc_result_free);
  const Eigen::Index n = rpc_result_n(r.get());
  const Eigen::Index k = rpc_result_rank(r.get());
  CholeskyResult res;
  res.approx.factor.resize(n, k);
  if (k > 0) {
    if (int st = rpc_result_factor_copy(r.get(), res.approx.factor.data(), n, RPC_COL_MAJOR))
      throw_status(st, rpc_last_error(dev.get()));
  }
  res.approx.pivots.resize(static_cast<std::size_t>(k));
  std::vector<int64_t> buf(static_cast<std::size_t>(k));
  rpc_result_pivots(r.get(), buf.data());
  for (Eigen::Index i = 0; i < k; ++i) res.approx.pivots[i] = static_cast<Eigen::Index>(buf[i]);
  res.approx.chol_factor.resize(k, k);
  if (k > 0) rpc_result_chol_copy(r.get(), res.approx.chol_factor.data());
  res.residual_diag.resize(n);
  rpc_result_residual_diag_copy(r.get(), res.residual_diag.data());
  const int64_t b = rpc_result_block_size(r.get());
  std::vector<int64_t> prop(static_cast<std::size_t>(b)), acc(static_cast<std::size_t>(b));
  for (int64_t t = 0; t < rpc_result_num_rounds(r.get()); ++t) {
    int64_t na = 0;
    rpc_result_round(r.get(), t, prop.data(), acc.data(), &na);
    RoundRecord rec;
    rec.proposed.assign(prop.begin(), prop.end());
    rec.accepted.assign(acc.begin(), acc.begin() + na);
    res.trace.rounds.push_back(std::move(rec));
  }
  res.trace.rank_exhausted = rpc_result_rank_exhausted(r.get()) != 0;
  res.trace.surplus = rpc_result_surplus(r.get());
  return res;
}

}  // namespace b200
}  // namespace rpchol

#endif  // RPCHOL_B200_HPP
