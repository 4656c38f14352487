/*
 * rpc_oracle.h — CPU restatement of the reference accelerated RPCholesky path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 library
 * (paper_2410_03969_b200/csrc).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path never links or calls anything in oracle/.
 *
 * It restates, function by function, the reference headers under
 * /root/reference/proj/include/rpchol (file:line cited at each definition in
 * rpc_oracle.c).  Pinning: SplitMix64 known-answer values (tests/golden), the
 * closed-form kernel values of test_kernel_oracle.cpp, the property suites of
 * test_rpcholesky.cpp, and the reference's own headers compiled here against a
 * minimal Eigen-API shim (oracle/_ref, see oracle/Makefile) — see DESIGN.md §3.
 *
 * Storage conventions follow the reference: matrices are column-major doubles
 * (Eigen::MatrixXd default), indices are int64 (Eigen::Index).
 */
#ifndef RPC_ORACLE_H
#define RPC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes mirror the reference exception classes. */
enum {
  RPO_OK = 0,
  RPO_EINVAL = 1,   /* std::invalid_argument */
  RPO_ERANGE = 2,   /* std::out_of_range */
  RPO_ENUMERIC = 3, /* std::runtime_error */
  RPO_ENOMEM = 4
};

enum { RPO_KERNEL_GAUSSIAN = 0, RPO_KERNEL_L1LAPLACE = 1, RPO_KERNEL_MATERN32 = 2, RPO_KERNEL_MATERN52 = 3 };
enum { RPO_DIST_DIRECT = 0, RPO_DIST_GRAM = 1 };
enum { RPO_MODE_FIXED_ROUNDS = 0, RPO_MODE_UNTIL_RANK = 1 };

/* ---- rng.hpp ---------------------------------------------------------- */
uint64_t rpo_splitmix64_draw(uint64_t seed, uint64_t n); /* n-th next_u64(), 0-based */
double rpo_u01(uint64_t z);                              /* next_double() mapping */
void rpo_cumulative_sums(const double* w, int64_t n, double* out);
int rpo_sample_discrete(const double* cumsum, int64_t n, double u01, int64_t* idx);
/* Decision-margin instrumentation (not in the reference; see rpc_oracle.c). */
void rpo_margins_reset(int on);
void rpo_margins_get(double* min_draw, double* min_sweep, int64_t* n_draws, int64_t* n_decisions);

/* ---- oracle.hpp ------------------------------------------------------- */
/* A PSD oracle: either a kernel over X (N x d, column-major) or a dense
 * N x N column-major matrix (DenseOracle, used by the ported algorithm tests). */
typedef struct {
  int is_dense;
  int64_t n;
  /* kernel oracle */
  const double* x; /* N x d col-major */
  int64_t d;
  int kind;
  double sigma;
  int dist_mode;
  double* sq_norms; /* owned, length N (kernel oracle ctor, oracle.hpp:252) */
  /* dense oracle */
  const double* a; /* N x N col-major */
  int n_threads;
} rpo_oracle;

int rpo_oracle_kernel(rpo_oracle* o, const double* x, int64_t n, int64_t d, int kind,
                      double sigma, int dist_mode, int n_threads);
int rpo_oracle_dense(rpo_oracle* o, const double* a, int64_t n);
void rpo_oracle_free(rpo_oracle* o);
/* out: nr x nc column-major */
int rpo_submatrix(const rpo_oracle* o, const int64_t* rows, int64_t nr, const int64_t* cols,
                  int64_t nc, double* out);

/* ---- rpcholesky.hpp --------------------------------------------------- */
/* Rejection sweep on an in/out b x b column-major block h (destroyed).  The
 * b accept draws are SplitMix64 draws [draw0, draw0 + b) of `seed`.
 * accepted/positions: length >= b; chol: length >= b*b, m x m column-major. */
int rpo_rejection_sweep(double* h, int64_t b, const int64_t* proposals, uint64_t seed,
                        uint64_t draw0, int64_t* accepted, int64_t* positions, int64_t* m,
                        double* chol);

typedef struct {
  int64_t block_size;
  int mode;
  int64_t rounds;
  int64_t target_rank;
  uint64_t seed;
  double stop_tol;
} rpo_run_config;

typedef struct {
  int64_t n;
  int64_t rank;          /* kcur at exit */
  double* factor;        /* n x rank col-major */
  int64_t* pivots;       /* rank */
  double* chol;          /* rank x rank col-major lower */
  double* residual_diag; /* n */
  int64_t n_rounds;
  int64_t block_size;
  int64_t* proposed;       /* n_rounds x b (row per round) */
  int64_t* accepted_count; /* n_rounds */
  int rank_exhausted;
  int64_t surplus;
  double captured_sq;
} rpo_result;

int rpo_accelerated_rpcholesky(const rpo_oracle* o, const rpo_run_config* cfg,
                               rpo_result* res);
/* Run only rounds [0, max_rounds) — bounded CPU-baseline samples. */
int rpo_accelerated_rpcholesky_bounded(const rpo_oracle* o, const rpo_run_config* cfg,
                                       int64_t max_rounds, rpo_result* res);
/* accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485): res->factor is NULL, res->chol
 * is the k x k L of the pivot block, res->rank = |pivots|. */
int rpo_accelerated_rpcholesky_lowmem(const rpo_oracle* o, const rpo_run_config* cfg,
                                      rpo_result* res);
/* block_rpcholesky (rpcholesky.hpp:268-333) and simple_rpcholesky (206-246); the PivotTrace
 * "accepted" lists are the kept (sorted, distinct) proposals. */
int rpo_block_rpcholesky(const rpo_oracle* o, const rpo_run_config* cfg, rpo_result* res);
int rpo_simple_rpcholesky(const rpo_oracle* o, int64_t k, uint64_t seed, rpo_result* res);
void rpo_result_free(rpo_result* res);
void rpo_free(void* p); /* one buffer taken out of a result */
double rpo_relative_trace_error(const rpo_oracle* o, const double* factor, int64_t n,
                                int64_t k);
const char* rpo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
