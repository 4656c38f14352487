// krr.cu — kernel ridge regression on the device (krr.hpp): the consumer of the
// factor that accelerated_rpcholesky leaves in HBM.
//
//   kernel_matvec  krr.hpp:143-162   A V without forming A.  One vector (every PCG step):
//                                    the symmetric product (symv.cu) generates each
//                                    1024 x 1024 block of the lower block triangle once and
//                                    uses it for A v and A^T v — N^2/2 kernel entries.  Up to
//                                    8 vectors (or RPC_KRR_GENERIC=1): the low-memory update
//                                    kernel in product mode (lowmem_impl.cuh), N^2 entries.
//                                    Kernel tiles are regenerated in registers (Gram on DMMA +
//                                    exp, or l1 distances on the FP64 cores); no N^2 storage.
//   Preconditioner krr.hpp:30-70     P = F F^T + mu I through Woodbury on the device-resident
//                                    F: core = F^T F + mu I by a DMMA SYRK, its blocked
//                                    Cholesky and the solves with it (krr_core.cu, no
//                                    library); apply_inverse is two HBM-bound F passes
//                                    (deterministic) around that solve.
//   pcg_solve      krr.hpp:87-123    textbook PCG, every vector on the device; one 24-byte
//                                    status read per iteration feeds the residual history.
//   fit_krr        krr.hpp:177-224   centre targets, accelerated_rpcholesky (UntilRank
//                                    min(rank, N), default distance mode), preconditioner,
//                                    PCG on (A + mu I) beta = y.
//   predict        krr.hpp:227-250   cross block query x training in product mode (no
//                                    same-index pin: different point sets) + target mean.
//
// Every reduction runs over a fixed partition of the rows and is summed in a fixed order,
// so results are bit-reproducible run to run.
#include <memory>

#include "runtime.h"

namespace rpcb_rt {

namespace {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs: fixed partition for every reduction
constexpr int kRedThreads = 256;

// ---- small device kernels ---------------------------------------------------
__global__ void records_kernel(const double* __restrict__ X, const double* __restrict__ sqn,
                               int64_t n, int64_t dpad, int64_t prec, double* __restrict__ rec) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  double* r = rec + i * prec;
  if (threadIdx.x == 0) {
    r[0] = (double)i;
    r[1] = sqn[i];
  }
  for (int64_t j = threadIdx.x; j < dpad; j += blockDim.x) r[2 + j] = X[i * dpad + j];
}

// Fixed row partition: block b owns rows [b * chunk, (b + 1) * chunk).
__device__ __forceinline__ void block_rows(int64_t n, int64_t& r0, int64_t& r1) {
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  r0 = (int64_t)blockIdx.x * chunk;
  r1 = r0 + chunk < n ? r0 + chunk : n;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum_xor(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  __syncthreads();
  return s;
}

// partial[b] = sum over block rows of a[i] * b[i]  (b == nullptr: a[i])
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   int64_t n, double* __restrict__ partial) {
  __shared__ double sh[32];
  int64_t r0, r1;
  block_rows(n, r0, r1);
  double s = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) s += b ? a[i] * b[i] : a[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out[slot] = sum of partial[0 .. nb) in order (one thread: fixed order)
__global__ void finish_kernel(const double* __restrict__ partial, int nb, double* out, int slot) {
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s += partial[i];
  out[slot] = s;
}

// y = t - mean, mean = s[0] / n  (Eigen: targets.array() - targets.mean())
__global__ void center_kernel(const double* __restrict__ t, int64_t n, const double* s,
                              double* __restrict__ y) {
  const double mean = s[0] / (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = t[i] - mean;
}

enum { S_RZ = 0, S_DENOM = 1, S_RR = 2, S_RU = 3, S_RZN = 4, S_MISC = 5 };

// if denom > 0: alpha = rz / denom, x += alpha p, r -= alpha ap; partials of ||r||^2 and
// ||r + mu x||^2 (krr.hpp:102-109)
__global__ void pcg_update_kernel(double* __restrict__ x, double* __restrict__ r,
                                  const double* __restrict__ p, const double* __restrict__ ap,
                                  int64_t n, const double* s, double mu,
                                  double* __restrict__ part_rr, double* __restrict__ part_ru) {
  __shared__ double sh[32];
  const double denom = s[S_DENOM];
  const bool go = denom > 0.0;
  const double alpha = go ? s[S_RZ] / denom : 0.0;
  int64_t r0, r1;
  block_rows(n, r0, r1);
  double rr = 0.0, ru = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double xi = x[i], ri = r[i];
    if (go) {
      xi += alpha * p[i];
      ri -= alpha * ap[i];
      x[i] = xi;
      r[i] = ri;
    }
    rr += ri * ri;
    const double t = ri + mu * xi;
    ru += t * t;
  }
  rr = block_sum(rr, sh);
  ru = block_sum(ru, sh);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = rr;
    part_ru[blockIdx.x] = ru;
  }
}

// p = z + (rz_next / rz) p   (krr.hpp:119-120)
__global__ void pcg_direction_kernel(double* __restrict__ p, const double* __restrict__ z,
                                     int64_t n, const double* s) {
  const double beta = s[S_RZN] / s[S_RZ];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

__global__ void roll_kernel(double* s) { s[S_RZ] = s[S_RZN]; }

__global__ void copy_kernel(const double* __restrict__ a, double* __restrict__ b, int64_t n,
                            double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = scale == 1.0 ? a[i] : a[i] / scale;
}

// Woodbury, step 1: partial[b][j] = sum over block rows of F[i][j] r[i]  (F^T r)
__global__ void ft_r_partial_kernel(const double* __restrict__ F, int64_t ldf, int64_t n, int k,
                                    const double* __restrict__ r, double* __restrict__ part) {
  int64_t r0, r1;
  block_rows(n, r0, r1);
  for (int j0 = 0; j0 < k; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    double s = 0.0;
    if (j < k)
      for (int64_t i = r0; i < r1; ++i) s += F[i * ldf + j] * r[i];
    if (j < k) part[(int64_t)blockIdx.x * k + j] = s;
  }
}

__global__ void ft_r_finish_kernel(const double* __restrict__ part, int nb, int k,
                                   double* __restrict__ t) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * k + j];
  t[j] = s;
}

// Woodbury, step 3: z = (r - F c) / mu, one warp per row (lanes stride the k columns,
// butterfly reduction: fixed order)
__global__ void woodbury_z_kernel(const double* __restrict__ F, int64_t ldf, int64_t n, int k,
                                  const double* __restrict__ c, const double* __restrict__ r,
                                  double mu, double* __restrict__ z) {
  extern __shared__ double sc[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) sc[j] = c[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const double* f = F + i * ldf;
    double s = 0.0;
    for (int j = lane; j < k; j += 32) s += f[j] * sc[j];
    s = warp_sum_xor(s);
    if (lane == 0) z[i] = (r[i] - s) / mu;
  }
}

// The symmetric product for one vector over n training points: from 16 super-blocks (enough
// units to fill the GPU) up to a 4 GB partial buffer (n ~ 7e5; beyond that the generic
// product, which needs no scratch).  RPC_KRR_GENERIC=1 forces the generic one (A/B runs).
bool use_symv(int64_t n) {
  static const bool generic = std::getenv("RPC_KRR_GENERIC") != nullptr;
  return !generic && n >= 16384 && symv_scratch_doubles(n) * 8 <= ((int64_t)4 << 30);
}

// X (host, any layout) -> packed device points [n][dpad] + norms; rejects non-finite.
void upload_points(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int layout,
                   int64_t dpad, DBuf& X, DBuf& sqn) {
  cudaStream_t st = ctx->stream;
  X = DBuf(ctx, sizeof(double) * n * dpad);
  sqn = DBuf(ctx, sizeof(double) * n);
  DBuf raw(ctx, sizeof(double) * n * d), bad(ctx, sizeof(int));
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  h2d_points(raw.p, x, n, d, ldx, layout, st);
  launch_pack_points(raw.as<double>(), n, (int)d, layout == RPC_ROW_MAJOR ? d : n,
                     layout == RPC_ROW_MAJOR, dpad, X.as<double>(), sqn.as<double>(),
                     bad.as<int>(), st);
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hbad) raise(RPC_EINVAL, "DataMatrix: non-finite entry");
}

}  // namespace

// A(R, S) W^T in product mode: rows = packed points (X, sqn), columns = point records.
void kernel_product(rpc_ctx* ctx, const double* X, const double* sqn, int64_t n_rows, int64_t dpad,
                    int64_t d, const double* rec, int64_t prec, int64_t n_cols, const double* W,
                    int64_t ldw, int m, int kind, int kfun, double kscale, int pin, double* out,
                    int64_t ld_out, const double* add_vec, double add_coef, double add_const) {
  LowmemParams lp{};
  lp.X = X;
  lp.dpad = dpad;
  lp.dchunks = (int)(dpad / 16);
  lp.d = (int)d;
  lp.sqn = sqn;
  lp.u = nullptr;
  lp.n_loc = n_rows;
  lp.row0 = 0;
  lp.piv = rec;
  lp.prec = prec;
  lp.W = W;
  lp.ldw = ldw;
  lp.m = m;
  lp.kold = (int)n_cols;  // no triangular structure in W
  lp.knew = (int)n_cols;
  lp.kind = kind;
  lp.kfun = kfun;
  lp.escale = kscale;
  lp.tile_g2 = nullptr;
  lp.out_mode = 1;
  lp.out = out;
  lp.ld_out = ld_out;
  lp.add_vec = add_vec;
  lp.add_coef = add_coef;
  lp.add_const = add_const;
  lp.pin = pin;
  const int bm = launch_lowmem(lp, ctx->stream);
  if (bm < 0) raise(RPC_ECUDA, "kernel product launch failed (code " + std::to_string(bm) + ")");
  dbg(ctx->stream, "kernel product");
}

}  // namespace rpcb_rt

using namespace rpcb_rt;

struct rpc_krr {
  rpc_ctx* ctx = nullptr;
  int64_t n = 0, d = 0, dpad = 0, prec = 0;
  int kind = 0, kfun = 0;
  double sigma = 1.0, kscale = 0.0, mu = 0.0, mean = 0.0;
  DBuf X, sqn, rec, coef;
  int64_t iterations = 0;
  bool converged = false;
  std::vector<double> rel, rel_unreg;
  std::vector<int64_t> pivots;
};

namespace {

int kind_of(rpc_kernel_spec k, int& mode_out) {
  // default_distance_mode (oracle.hpp:39-42): Gram trick for the Gaussian, direct for l1
  int kind;
  rpc_run_config dummy{1, RPC_UNTIL_RANK, 0, 1, 0, 0.0, 0};
  k.distance_mode = RPC_DIST_DEFAULT;
  validate(1, 1, k, dummy, kind);
  mode_out = RPC_DIST_DEFAULT;
  return kind;
}

}  // namespace

extern "C" {

int rpc_kernel_matvec(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int layout,
                      rpc_kernel_spec kspec, const double* v, int64_t nrhs, double* out) {
  if (!ctx) return fail(nullptr, RPC_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded(ctx, [&] {
    int kind = 0;
    rpc_run_config cfg{1, RPC_UNTIL_RANK, 0, 1, 0, 0.0, 0};
    validate(n, d, kspec, cfg, kind);
    double kscale = 0.0;
    const int kfun = kernel_fun(kspec, &kscale);
    if (nrhs < 1 || nrhs > 8) raise(RPC_EINVAL, "kernel_matvec: this build supports 1..8 right-hand sides");
    if (round_up(d, 16) > 128) raise(RPC_EINVAL, "kernel_matvec: this build supports d <= 128");
    if (ldx < (layout == RPC_ROW_MAJOR ? d : n)) raise(RPC_EINVAL, "leading dimension too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t dpad = round_up(d, 16), prec = 2 + dpad, ldv = round_up(n, 16);
    DBuf X, sqn;
    upload_points(ctx, x, n, d, ldx, layout, dpad, X, sqn);
    DBuf rec(ctx, sizeof(double) * n * prec), W(ctx, sizeof(double) * nrhs * ldv),
        o(ctx, sizeof(double) * n * nrhs);
    records_kernel<<<(unsigned)n, 64, 0, st>>>(X.as<double>(), sqn.as<double>(), n, dpad, prec,
                                               rec.as<double>());
    // V (n x nrhs column-major) is W^T row-major with rows padded to ldv
    CK(cudaMemcpy2DAsync(W.p, ldv * 8, v, n * 8, n * 8, nrhs, cudaMemcpyHostToDevice, st));
    DBuf sym;
    bool done = false;
    if (nrhs == 1 && use_symv(n)) {  // one vector: symmetric blocks, each generated once
      sym = DBuf(ctx, sizeof(double) * symv_scratch_doubles(n));
      done = launch_symv(X.as<double>(), dpad, (int)d, sqn.as<double>(), rec.as<double>(), prec,
                         W.as<double>(), ldv, n, kind, kfun, kscale, sym.as<double>(), nullptr,
                         0.0, 0.0, o.as<double>(), st);
    }
    if (!done)
      kernel_product(ctx, X.as<double>(), sqn.as<double>(), n, dpad, d, rec.as<double>(), prec, n,
                     W.as<double>(), ldv, (int)nrhs, kind, kfun, kscale, 1, o.as<double>(), nrhs,
                     nullptr, 0.0, 0.0);
    // out: n x nrhs column-major <- o row-major [n][nrhs]
    if (nrhs == 1) {
      CK(cudaMemcpyAsync(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    } else {
      std::vector<double> h((size_t)(n * nrhs));
      CK(cudaMemcpyAsync(h.data(), o.p, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < nrhs; ++j) out[j * n + i] = h[(size_t)(i * nrhs + j)];
    }
    CK(cudaStreamSynchronize(st));
  });
}

int rpc_krr_fit(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int layout,
                rpc_kernel_spec kspec, const double* targets, double mu, int64_t precond_rank,
                rpc_run_config cfg, double tol, int64_t max_iters, rpc_krr** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  *out = nullptr;
  std::unique_ptr<rpc_krr> m(new rpc_krr());
  int rc = guarded(ctx, [&] {
    if (ctx->nshards() != 1) raise(RPC_EINVAL, "fit_krr: single-shard contexts only in this build");
    int dmode = 0;
    const int kind = kind_of(kspec, dmode);
    if (n < 1 || d < 1) raise(RPC_EINVAL, "DataMatrix: need at least one point and one dimension");
    if (!(mu > 0.0)) raise(RPC_EINVAL, "fit_krr: mu must be > 0");
    if (!(tol > 0.0)) raise(RPC_EINVAL, "pcg_solve: tol must be > 0");
    if (round_up(d, 16) > 128) raise(RPC_EINVAL, "fit_krr: this build supports d <= 128");
    if (ldx < (layout == RPC_ROW_MAJOR ? d : n)) raise(RPC_EINVAL, "leading dimension too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    m->ctx = ctx;
    m->n = n;
    m->d = d;
    m->dpad = round_up(d, 16);
    m->prec = 2 + m->dpad;
    m->kind = kind;
    m->sigma = kspec.sigma;
    m->kfun = kernel_fun(kspec, &m->kscale);
    m->mu = mu;

    // ---- low-rank preconditioner: accelerated_rpcholesky, UntilRank(min(rank, N)) ----
    std::unique_ptr<rpc_result> res;
    int64_t k = 0;
    if (precond_rank > 0) {
      rpc_run_config c2 = cfg;
      c2.mode = RPC_UNTIL_RANK;
      c2.target_rank = std::min(precond_rank, n);
      // (the preconditioner keeps the FP64 DMMA residual: PCG iteration counts follow the
      // reference's to +-1 with it, and moved by 3 on a fixture with the int8 digit path)
      c2.flags = RPC_FLAG_FP64_RESIDUAL;
      rpc_kernel_spec ks = kspec;
      ks.distance_mode = RPC_DIST_DEFAULT;
      res.reset(new rpc_result());
      {
        std::lock_guard<std::mutex> lk(ctx->mu);
        run_factorization(ctx, x, false, n, d, ldx, layout, ks, c2, res.get());
      }
      k = res->kcur;
      m->pivots = res->pivots;
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    upload_points(ctx, x, n, d, ldx, layout, m->dpad, m->X, m->sqn);
    m->rec = DBuf(ctx, sizeof(double) * n * m->prec);
    records_kernel<<<(unsigned)n, 64, 0, st>>>(m->X.as<double>(), m->sqn.as<double>(), n, m->dpad,
                                               m->prec, m->rec.as<double>());

    // ---- targets: y = t - mean (krr.hpp:185-186) ----
    const int nb = (int)std::min<int64_t>(kRedBlocks, n);
    DBuf t(ctx, sizeof(double) * n), y(ctx, sizeof(double) * n), part(ctx, sizeof(double) * nb * 2),
        s(ctx, sizeof(double) * 8);
    CK(cudaMemsetAsync(s.p, 0, sizeof(double) * 8, st));
    CK(cudaMemcpyAsync(t.p, targets, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(t.as<double>(), nullptr, n, part.as<double>());
    finish_kernel<<<1, 1, 0, st>>>(part.as<double>(), nb, s.as<double>(), S_MISC);
    double* s_d = s.as<double>();
    center_kernel<<<nb, kRedThreads, 0, st>>>(t.as<double>(), n, s_d + S_MISC, y.as<double>());
    dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(y.as<double>(), y.as<double>(), n,
                                                   part.as<double>());
    finish_kernel<<<1, 1, 0, st>>>(part.as<double>(), nb, s_d, S_RR);
    double hs[8];
    CK(cudaMemcpyAsync(hs, s.p, sizeof(double) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    m->mean = hs[S_MISC] / (double)n;
    const double norm_y = std::sqrt(hs[S_RR]);
    m->coef = DBuf(ctx, sizeof(double) * round_up(n, 16));
    CK(cudaMemsetAsync(m->coef.p, 0, m->coef.bytes, st));
    if (norm_y == 0.0) {  // constant targets: centering absorbs everything (krr.hpp:201-206)
      m->converged = true;
      CK(cudaStreamSynchronize(st));
      return;
    }

    // ---- preconditioner core = F^T F + mu I, Cholesky (krr.hpp:33-44) ----
    const double* F = k > 0 ? res->shards[0].F.as<double>() : nullptr;
    const int64_t ldf = k > 0 ? res->ldf : 0;
    DBuf core, scratch, info, tvec, part_k;
    int64_t kc = 0;
    if (k > 0) {
      kc = core_dim((int)k);
      core = DBuf(ctx, sizeof(double) * kc * kc);
      scratch = DBuf(ctx, sizeof(double) * core_syrk_scratch_doubles((int)k));
      launch_core_syrk(F, ldf, n, (int)k, mu, core.as<double>(), scratch.as<double>(), st);
      info = DBuf(ctx, sizeof(int));
      CK(cudaMemsetAsync(info.p, 0, sizeof(int), st));
      launch_core_potrf(core.as<double>(), kc, info.as<int>(), st);
      int hinfo = 0;
      CK(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaGetLastError());
      if (hinfo != 0) raise(RPC_ENUMERIC, "Preconditioner: core factorization failed");
      scratch.release();
      tvec = DBuf(ctx, sizeof(double) * kc);
      CK(cudaMemsetAsync(tvec.p, 0, sizeof(double) * kc, st));  // padding stays 0
      part_k = DBuf(ctx, sizeof(double) * (size_t)nb * k);
    }
    const double pmu = k > 0 ? mu : 1.0;  // Preconditioner::identity() has mu = 1
    auto apply_inverse = [&](const double* r, double* z) {  // krr.hpp:47-51
      if (k == 0) {
        copy_kernel<<<nb, kRedThreads, 0, st>>>(r, z, n, pmu);
        return;
      }
      ft_r_partial_kernel<<<nb, 256, 0, st>>>(F, ldf, n, (int)k, r, part_k.as<double>());
      ft_r_finish_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(part_k.as<double>(), nb,
                                                                      (int)k, tvec.as<double>());
      launch_core_potrs(core.as<double>(), kc, tvec.as<double>(), st);
      woodbury_z_kernel<<<nb, 256, sizeof(double) * k, st>>>(F, ldf, n, (int)k, tvec.as<double>(),
                                                             r, mu, z);
    };
    if (k > 0) ensure_smem_attr((const void*)woodbury_z_kernel, (int)(sizeof(double) * k));

    // ---- PCG on (A + mu I) beta = y (krr.hpp:87-123) ----
    const int64_t ldv = round_up(n, 16);
    DBuf r(ctx, sizeof(double) * n), z(ctx, sizeof(double) * n), p(ctx, sizeof(double) * ldv),
        ap(ctx, sizeof(double) * n), prr(ctx, sizeof(double) * nb), pru(ctx, sizeof(double) * nb);
    double* xb = m->coef.as<double>();
    CK(cudaMemcpyAsync(r.p, y.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    apply_inverse(r.as<double>(), z.as<double>());
    CK(cudaMemsetAsync(p.p, 0, p.bytes, st));
    CK(cudaMemcpyAsync(p.p, z.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(r.as<double>(), z.as<double>(), n,
                                                   part.as<double>());
    finish_kernel<<<1, 1, 0, st>>>(part.as<double>(), nb, s_d, S_RZ);
    double* hst = static_cast<double*>(ctx->pinned(sizeof(double) * 8));
    DBuf sym;
    if (use_symv(n)) sym = DBuf(ctx, sizeof(double) * symv_scratch_doubles(n));
    for (int64_t it = 0; it < max_iters; ++it) {
      // ap = A p + mu p  (fused kernel regeneration + tensor-core / FMA product; the
      // symmetric form generates each off-diagonal block once for A p and A^T p)
      const bool done =
          sym.p && launch_symv(m->X.as<double>(), m->dpad, (int)d, m->sqn.as<double>(),
                               m->rec.as<double>(), m->prec, p.as<double>(), ldv, n, kind, m->kfun,
                               m->kscale, sym.as<double>(), p.as<double>(), mu, 0.0,
                               ap.as<double>(), st);
      if (!done)
        kernel_product(ctx, m->X.as<double>(), m->sqn.as<double>(), n, m->dpad, d,
                       m->rec.as<double>(), m->prec, n, p.as<double>(), ldv, 1, kind, m->kfun,
                       m->kscale, 1, ap.as<double>(), 1, p.as<double>(), mu, 0.0);
      dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(p.as<double>(), ap.as<double>(), n,
                                                     part.as<double>());
      finish_kernel<<<1, 1, 0, st>>>(part.as<double>(), nb, s_d, S_DENOM);
      pcg_update_kernel<<<nb, kRedThreads, 0, st>>>(xb, r.as<double>(), p.as<double>(),
                                                    ap.as<double>(), n, s_d, mu, prr.as<double>(),
                                                    pru.as<double>());
      finish_kernel<<<1, 1, 0, st>>>(prr.as<double>(), nb, s_d, S_RR);
      finish_kernel<<<1, 1, 0, st>>>(pru.as<double>(), nb, s_d, S_RU);
      // speculative next direction (discarded when this iteration stops the solve)
      apply_inverse(r.as<double>(), z.as<double>());
      dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(r.as<double>(), z.as<double>(), n,
                                                     part.as<double>());
      finish_kernel<<<1, 1, 0, st>>>(part.as<double>(), nb, s_d, S_RZN);
      pcg_direction_kernel<<<nb, kRedThreads, 0, st>>>(p.as<double>(), z.as<double>(), n, s_d);
      roll_kernel<<<1, 1, 0, st>>>(s_d);
      CK(cudaMemcpyAsync(hst, s.p, sizeof(double) * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaGetLastError());
      if (!(hst[S_DENOM] > 0.0)) break;  // loss of positive definiteness
      m->iterations = it + 1;
      const double rel = std::sqrt(hst[S_RR]) / norm_y;
      m->rel.push_back(rel);
      m->rel_unreg.push_back(std::sqrt(hst[S_RU]) / norm_y);
      if (rel < tol) {
        m->converged = true;
        break;
      }
    }
    CK(cudaStreamSynchronize(st));
  });
  if (rc) return rc;
  *out = m.release();
  return RPC_OK;
}

int64_t rpc_krr_iterations(const rpc_krr* m) { return m ? m->iterations : 0; }
int rpc_krr_converged(const rpc_krr* m) { return m ? (int)m->converged : 0; }
double rpc_krr_target_mean(const rpc_krr* m) { return m ? m->mean : 0.0; }
int64_t rpc_krr_precond_rank(const rpc_krr* m) { return m ? (int64_t)m->pivots.size() : 0; }

int rpc_krr_residuals(const rpc_krr* m, double* reg, double* unreg) {
  if (!m) return RPC_EINVAL;
  if (reg) std::copy(m->rel.begin(), m->rel.end(), reg);
  if (unreg) std::copy(m->rel_unreg.begin(), m->rel_unreg.end(), unreg);
  return RPC_OK;
}

int rpc_krr_precond_pivots(const rpc_krr* m, int64_t* out) {
  if (!m) return RPC_EINVAL;
  std::copy(m->pivots.begin(), m->pivots.end(), out);
  return RPC_OK;
}

int rpc_krr_coefficients(const rpc_krr* m, double* out) {
  if (!m) return RPC_EINVAL;
  rpc_ctx* ctx = m->ctx;
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaMemcpyAsync(out, m->coef.p, sizeof(double) * m->n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int rpc_krr_predict(const rpc_krr* m, const double* q, int64_t nq, int64_t d, int64_t ldq,
                    int layout, double* out) {
  if (!m) return RPC_EINVAL;
  rpc_ctx* ctx = m->ctx;
  return guarded(ctx, [&] {
    if (d != m->d) raise(RPC_EINVAL, "predict: query dimension mismatch");
    if (nq < 1) raise(RPC_EINVAL, "DataMatrix: need at least one point and one dimension");
    if (ldq < (layout == RPC_ROW_MAJOR ? d : nq)) raise(RPC_EINVAL, "leading dimension too small");
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DBuf Q, qsqn, o(ctx, sizeof(double) * nq);
    upload_points(ctx, q, nq, d, ldq, layout, m->dpad, Q, qsqn);
    // f(x) = sum_i beta_i kappa(x_i, x) + mean; query and training are different sets:
    // no same-index pin (oracle.hpp:149-166)
    kernel_product(ctx, Q.as<double>(), qsqn.as<double>(), nq, m->dpad, d, m->rec.as<double>(),
                   m->prec, m->n, m->coef.as<double>(), round_up(m->n, 16), 1, m->kind, m->kfun, m->kscale,
                   0, o.as<double>(), 1, nullptr, 0.0, m->mean);
    CK(cudaMemcpyAsync(out, o.p, sizeof(double) * nq, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

void rpc_krr_free(rpc_krr* m) {
  if (!m) return;
  if (m->ctx) {
    std::lock_guard<std::mutex> lk(m->ctx->mu);
    cudaStreamSynchronize(m->ctx->stream);
    m->X.release();
    m->sqn.release();
    m->rec.release();
    m->coef.release();
  }
  delete m;
}

}  // extern "C"
