/*
 * rpchol_gpu.h — C-ABI of the B200-native accelerated RPCholesky library
 * (librpchol_b200.so, built from paper_2410_03969_b200/csrc).
 *
 * Drop-in boundary for the reference hot path
 *   CholeskyResult rpchol::accelerated_rpcholesky(const PsdOracle&, const RunConfig&)
 *     /root/reference/proj/include/rpchol/rpcholesky.hpp:338-401
 * specialised to the implicit kernel oracle
 *   KernelOracle(DataMatrix X, KernelSpec{kind, sigma}, DistanceMode)
 *     /root/reference/proj/include/rpchol/oracle.hpp:243-258
 * Plain pointers and sizes only; no torch, no Eigen in any signature.  Every
 * entry point returns an rpc_status; rpc_last_error() gives the message, which
 * reuses the reference's exception strings where one exists.
 *
 * There is no CPU fallback: without a usable sm_100a device every compute entry
 * point fails with RPC_ECUDA.
 */
#ifndef RPCHOL_GPU_H
#define RPCHOL_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rpc_ctx rpc_ctx;
typedef struct rpc_result rpc_result;

/* Status codes <-> reference exception classes (rpchol_cli.cpp:26-28). */
typedef enum {
  RPC_OK = 0,
  RPC_EINVAL = 1,   /* std::invalid_argument */
  RPC_ERANGE = 2,   /* std::out_of_range */
  RPC_ENUMERIC = 3, /* std::runtime_error (numerical) */
  RPC_ECUDA = 4,    /* CUDA failure / no device */
  RPC_ENCCL = 5,    /* NCCL failure */
  RPC_ENOMEM = 6    /* device or host allocation failed */
} rpc_status;

/* KernelKind (kernels.hpp:20): every kind the reference's KernelOracle supports. */
typedef enum {
  RPC_KERNEL_GAUSSIAN = 0,
  RPC_KERNEL_L1LAPLACE = 1,
  RPC_KERNEL_MATERN32 = 2,
  RPC_KERNEL_MATERN52 = 3
} rpc_kernel_kind;
/* DistanceMode (oracle.hpp:37); DEFAULT = default_distance_mode (oracle.hpp:39-42). */
typedef enum { RPC_DIST_DIRECT = 0, RPC_DIST_GRAM = 1, RPC_DIST_DEFAULT = -1 } rpc_distance_mode;
/* RunConfig::Mode (rpcholesky.hpp:37). */
typedef enum { RPC_FIXED_ROUNDS = 0, RPC_UNTIL_RANK = 1 } rpc_run_mode;
typedef enum { RPC_COL_MAJOR = 0, RPC_ROW_MAJOR = 1 } rpc_layout;

/* KernelSpec (kernels.hpp:41-51) + the oracle's DistanceMode. */
typedef struct {
  int kind;          /* rpc_kernel_kind */
  double sigma;      /* bandwidth, > 0 and finite */
  int distance_mode; /* rpc_distance_mode */
} rpc_kernel_spec;

/* RunConfig (rpcholesky.hpp:36-67) plus B200 execution flags. */
enum {
  /* sequential cumulative_sums + upper_bound exactly as rng.hpp:67-96 over the global
     residual diagonal (gathered on every shard when sharded); slower */
  RPC_FLAG_REPLAY_SCAN = 1u,
  /* every round's residual GEMM on the FP64 DMMA path (no int8 tensor-core digit
     products) */
  RPC_FLAG_FP64_RESIDUAL = 2u
};
typedef struct {
  int64_t block_size;  /* b >= 1 (this build: b <= 1024; low-memory variant b <= 256) */
  int mode;            /* rpc_run_mode */
  int64_t rounds;      /* FixedRounds: t >= 1 */
  int64_t target_rank; /* UntilRank: k >= 1 */
  uint64_t seed;       /* SplitMix64 seed */
  double stop_tol;     /* 0 disables the early exit */
  uint32_t flags;
} rpc_run_config;

/* ---- context ------------------------------------------------------------ */
/* One GPU, one shard. */
int rpc_create(int device, rpc_ctx** out);
/* One GPU holding n_shards row shards with device-local collectives; produces
 * the same pivots and factor as an n_shards-GPU run (p-invariance testing). */
int rpc_create_virtual(int device, int n_shards, rpc_ctx** out);
/* One process per GPU: rank `rank` of `nranks`, NCCL communicator built from a
 * 128-byte ncclUniqueId produced by rpc_nccl_unique_id on one rank and shared
 * by the caller (e.g. over torch.distributed / MPI / files). */
int rpc_nccl_unique_id(void* id128);
int rpc_create_nccl(int device, const void* id128, int nranks, int rank, rpc_ctx** out);
/* One rank of an nranks-process job whose collectives the caller provides on the host
 * (e.g. torch.distributed over gloo, MPI): the library synchronises its stream, stages the
 * data through pinned memory and calls back.  Same protocol, results and p-invariance as
 * the NCCL context, at host-link speed — meant for CPU-transport jobs and for running
 * several ranks on one GPU in tests (the kernels never wait on another rank).
 * Callbacks return 0 on success; `ops` is copied, `user` must outlive the context. */
typedef struct {
  void* user;
  /* every rank contributes `bytes` from send; recv receives nranks * bytes, rank order */
  int (*allgather)(void* user, const void* send, void* recv, size_t bytes);
  /* in place: word i becomes the bitwise OR of word i over all ranks (the library only
   * reduces buffers in which at most one rank holds a non-zero word, so any exact
   * combine — OR, unsigned max — is valid) */
  int (*allreduce_or_u64)(void* user, uint64_t* buf, size_t count);
} rpc_host_collectives;
int rpc_create_hostcoll(int device, int nranks, int rank, const rpc_host_collectives* ops,
                        rpc_ctx** out);
void rpc_destroy(rpc_ctx* ctx);
/* Message of the last failing call on this thread (or on ctx when non-null). */
const char* rpc_last_error(const rpc_ctx* ctx);
/* Global shard layout of a run on N points: rows [row0, row0+nrows) are owned by
 * this process's shard `local` (0 unless virtual). */
int rpc_shard_rows(const rpc_ctx* ctx, int64_t n, int local, int64_t* row0, int64_t* nrows);

/* Host-only shard plan (no device needed): N points over n_shards global shards.
 * Rows are cut at multiples of the 4096-row scan chunk, so the chunk grid, and with
 * it every reduction order, is independent of the shard count (p-invariance).
 * Shard s owns rows [row0, row0+nrows) = global chunks [chunk0, chunk0+nchunks);
 * every shard reserves chunks_per_shard slots in the per-round allgathers. */
int rpc_plan_shards(int64_t n, int n_shards, int shard, int64_t* row0, int64_t* nrows,
                    int* chunk0, int* nchunks, int* chunks_per_shard);

/* ---- the hot path: accelerated_rpcholesky over a kernel oracle ----------- */
/* X: host N x d points (layout + leading dimension ldx).  Every rank passes the
 * same full X; each uploads only its own rows. */
int rpc_accelerated_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                               int layout, rpc_kernel_spec kernel, rpc_run_config cfg,
                               rpc_result** out);
/* Same with the points already resident on the device: x_dev holds this
 * process's shard rows [row0, row0+nrows) (see rpc_shard_rows) in `layout`
 * with leading dimension ldx.  No host<->device traffic besides per-round
 * status words. */
int rpc_accelerated_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                      int64_t ldx, int layout, rpc_kernel_spec kernel,
                                      rpc_run_config cfg, rpc_result** out);

/* Same, with the factor delivered to host memory while the rounds run: factor_out is
 * column-major, element (i, j) at factor_out[j * ld_out + i] for the global rows i this
 * process owns (ld_out >= its row count; pass base - row0 for a rank-local buffer), with
 * cols_out >= min(N, k + b) (FixedRounds:
 * min(N, t b)) columns; on return its first rpc_result_rank() columns hold this process's
 * rows of F.  Each round's finished columns are transposed and copied on a second stream,
 * overlapping the next rounds (the buffer is page-locked for the call unless it already is). */
int rpc_accelerated_rpcholesky_into(rpc_ctx* ctx, const double* x, int64_t n, int64_t d,
                                    int64_t ldx, int layout, rpc_kernel_spec kernel,
                                    rpc_run_config cfg, double* factor_out, int64_t ld_out,
                                    int64_t cols_out, rpc_result** out);

/* ---- low-memory variant ------------------------------------------------- */
/* accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485; LowMemResult 114-119):
 * same pivots, trace and stopping rules as the standard call; keeps O(N + k^2)
 * state (X, u, pivots, L, L^{-1}) and never stores the N x k factor.  The result
 * handle answers rank / pivots / chol_copy / residual_diag_copy / round /
 * rank_exhausted / surplus / captured_sq; rpc_result_factor_copy fails with
 * RPC_EINVAL and rpc_result_factor_device returns NULL.  This build: d <= 128. */
int rpc_accelerated_rpcholesky_lowmem(rpc_ctx* ctx, const double* x, int64_t n, int64_t d,
                                      int64_t ldx, int layout, rpc_kernel_spec kernel,
                                      rpc_run_config cfg, rpc_result** out);
int rpc_accelerated_rpcholesky_lowmem_device(rpc_ctx* ctx, const double* x_dev, int64_t n,
                                             int64_t d, int64_t ldx, int layout,
                                             rpc_kernel_spec kernel, rpc_run_config cfg,
                                             rpc_result** out);
int rpc_result_is_lowmem(const rpc_result* r);

/* ---- block and simple RPCholesky (the paper's baselines) ------------------ */
/* block_rpcholesky (rpcholesky.hpp:268-333): per round b proposals (draws [b r, b r + b)),
 * every distinct one kept (sorted), the kept block Cholesky-factored (one retry with a
 * 64 eps tr(A)/N diagonal shift, then RPC_ENUMERIC) and eliminated.  Same result handle. */
int rpc_block_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                         int layout, rpc_kernel_spec kernel, rpc_run_config cfg, rpc_result** out);
int rpc_block_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                int64_t ldx, int layout, rpc_kernel_spec kernel,
                                rpc_run_config cfg, rpc_result** out);
/* simple_rpcholesky (rpcholesky.hpp:206-246): k sequential pivots, one draw each; a
 * non-positive residual pivot sets rank_exhausted.  flags: RPC_FLAG_REPLAY_SCAN. */
int rpc_simple_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                          int layout, rpc_kernel_spec kernel, int64_t k, uint64_t seed,
                          uint32_t flags, rpc_result** out);
int rpc_simple_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                 int64_t ldx, int layout, rpc_kernel_spec kernel, int64_t k,
                                 uint64_t seed, uint32_t flags, rpc_result** out);

/* ---- result (CholeskyResult, rpcholesky.hpp:106-110) --------------------- */
int64_t rpc_result_n(const rpc_result* r);
int64_t rpc_result_rank(const rpc_result* r); /* factor columns = |pivots| */
int rpc_result_pivots(const rpc_result* r, int64_t* out); /* rank entries */
/* Factor rows owned by this process: writes rows [row0, row0+nrows) of the
 * N x rank factor into out (global row indexing; ld = leading dimension). */
int rpc_result_factor_copy(const rpc_result* r, double* out, int64_t ld, int layout);
/* chol_factor: rank x rank lower triangle, column-major (rpcholesky.hpp:140-145). */
int rpc_result_chol_copy(const rpc_result* r, double* out);
/* residual_diag rows owned by this process (global indexing into out[N]). */
int rpc_result_residual_diag_copy(const rpc_result* r, double* out);
int64_t rpc_result_num_rounds(const rpc_result* r);
int64_t rpc_result_block_size(const rpc_result* r);
/* PivotTrace rounds (rpcholesky.hpp:78-104): proposed has block_size entries;
 * accepted receives up to block_size entries, *n_accepted its count. */
int rpc_result_round(const rpc_result* r, int64_t round, int64_t* proposed, int64_t* accepted,
                     int64_t* n_accepted);
int rpc_result_rank_exhausted(const rpc_result* r);
int64_t rpc_result_surplus(const rpc_result* r);
double rpc_result_captured_sq(const rpc_result* r);
/* relative_trace_error (rpcholesky.hpp:577-583), from the device-resident factor. */
double rpc_result_relative_trace_error(const rpc_result* r);
/* Device-resident factor of this process's (first) shard: row-major, ld = *ldf. */
const double* rpc_result_factor_device(const rpc_result* r, int64_t* ldf, int64_t* row0,
                                       int64_t* nrows);

/* write_rpcf (io.hpp:218-256) from the device-resident result: byte-identical to the
 * reference's file for the same factor, pivots and chol_factor.  Under NCCL every rank
 * calls it with the same path on a shared filesystem; each writes its own rows. */
int rpc_result_write_rpcf(const rpc_result* r, const char* path);
/* write_pivot_trace_csv (io.hpp:336-350). */
int rpc_result_write_trace_csv(const rpc_result* r, const char* path);

typedef struct {
  double factorize_ms;     /* device time, first kernel to factor complete (CUDA events) */
  double upload_ms;        /* X host->device + packing */
  double update_ms;        /* sum over rounds of the fused K5+K6 update kernel(s) */
  double update_flops;     /* algorithmic FP64 flops of those launches */
  double update_bytes;     /* algorithmic HBM bytes of those launches */
  int64_t update_launches; /* update-kernel launches */
  int64_t kernel_launches; /* all kernels launched by the factorization */
  double host_total_ms;    /* host wall time of the whole call */
  double host_setup_ms;    /* ... allocation, upload, packing, validation */
  double host_loop_ms;     /* ... the round loop */
  double host_final_ms;    /* ... finalisation (chol gather, bookkeeping) */
  /* rounds whose residual GEMM F B'^T ran on the tensor cores (int8 digit planes, i8gemm.cu;
   * included in update_ms / update_flops above): */
  double tc_ms;            /* device time of those launches (digit planes of B' + GEMM) */
  double tc_int8_ops;      /* int8 tensor-core operations issued (2 per MAC, padded shapes) */
  double tc_fp64_flops;    /* the FP64 flops of the GEMMs they replaced (2 N m kcur) */
  double tc_slice_ms;      /* device time appending F's columns to its digit planes */
} rpc_timing;
int rpc_result_timing(const rpc_result* r, rpc_timing* t);
void rpc_result_free(rpc_result* r);

/* ---- component entry points (reference public functions) ---------------- */
/* KernelOracle::columns (oracle.hpp:188-191) through the standalone K5 kernel:
 * out (N x m, column-major, ld) = A(:, cols).  *device_ms = kernel time. */
int rpc_kernel_columns(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                       int layout, rpc_kernel_spec kernel, const int64_t* cols, int64_t m,
                       double* out, int64_t ld_out, double* device_ms);
/* bench_column_throughput (experiment.hpp:344-387): ~1000 columns drawn as
 * SplitMix64(seed).next_u64() % N, generated on the device in blocks of each requested
 * size (one standalone K5 launch per block of <= 256 columns, output kept in HBM), for the
 * Direct and (Gaussian only) GramTrick modes.  rows needs 2 * n_sizes entries; wall_ms
 * is device time (CUDA events) after one warm-up pass; output_gbs = 8 N columns / time. */
typedef struct {
  int64_t block_size;
  int distance_mode; /* rpc_distance_mode */
  int64_t columns;
  double wall_ms;
  double columns_per_sec;
  double output_gbs; /* kernel-col GB/s (BASELINE metric) */
} rpc_throughput_row;
int rpc_bench_column_throughput(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                                int layout, rpc_kernel_spec kernel, const int64_t* block_sizes,
                                int n_sizes, uint64_t seed, rpc_throughput_row* rows,
                                int* n_rows);
/* b draws of sample_discrete (rng.hpp:80-96) against cumulative_sums(u), using
 * SplitMix64(seed) draws [draw0, draw0+b).  replay != 0: sequential scan. */
int rpc_sample_discrete(rpc_ctx* ctx, const double* u, int64_t n, int64_t b, uint64_t seed,
                        uint64_t draw0, int replay, int64_t* out);
/* rejection_sample_submatrix (rpcholesky.hpp:167-201): h is b x b column-major;
 * accept draws are SplitMix64(seed) draws [draw0, draw0+b).  chol: m x m
 * column-major (capacity b*b). */
int rpc_rejection_sweep(rpc_ctx* ctx, const double* h, int64_t b, const int64_t* proposals,
                        uint64_t seed, uint64_t draw0, int64_t* accepted, int64_t* positions,
                        int64_t* m, double* chol);

/* ---- kernel ridge regression (krr.hpp) ------------------------------------ */
/* kernel_matvec (krr.hpp:143-162): out (n x nrhs, column-major) = A V for V (n x nrhs,
 * column-major), A the kernel matrix of X, never formed.  nrhs in [1, 8]; d <= 128. */
int rpc_kernel_matvec(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                      int layout, rpc_kernel_spec kernel, const double* v, int64_t nrhs,
                      double* out);
typedef struct rpc_krr rpc_krr;
/* fit_krr (krr.hpp:177-224): centred targets, accelerated_rpcholesky preconditioner of
 * rank min(precond_rank, n) (0 = plain CG; cfg supplies block size and seed; the kernel
 * uses default_distance_mode, oracle.hpp:39-42), Woodbury preconditioner (krr.hpp:30-70),
 * PCG on (A + mu I) beta = y to relative residual tol (krr.hpp:87-123).  Errors:
 * RPC_EINVAL for mu <= 0, tol <= 0, bad shapes; RPC_ENUMERIC if the core factorization
 * fails.  Single-shard contexts. */
int rpc_krr_fit(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int layout,
                rpc_kernel_spec kernel, const double* targets, double mu, int64_t precond_rank,
                rpc_run_config cfg, double tol, int64_t max_iters, rpc_krr** out);
int64_t rpc_krr_iterations(const rpc_krr* m);  /* PcgReport::iterations */
int rpc_krr_converged(const rpc_krr* m);       /* PcgReport::converged */
/* PcgReport::relative_residuals / relative_residuals_unreg (iterations entries each) */
int rpc_krr_residuals(const rpc_krr* m, double* reg, double* unreg);
int rpc_krr_coefficients(const rpc_krr* m, double* out); /* KrrModel::coefficients (n) */
double rpc_krr_target_mean(const rpc_krr* m);            /* KrrModel::target_mean */
int64_t rpc_krr_precond_rank(const rpc_krr* m);          /* KrrFitResult::preconditioner rank */
int rpc_krr_precond_pivots(const rpc_krr* m, int64_t* out);
/* predict (krr.hpp:227-250): out[nq] = sum_i beta_i kappa(x_i, q) + target mean */
int rpc_krr_predict(const rpc_krr* m, const double* q, int64_t nq, int64_t d, int64_t ldq,
                    int layout, double* out);
void rpc_krr_free(rpc_krr* m);

#ifdef __cplusplus
}
#endif
#endif /* RPCHOL_GPU_H */
