// kernels.h — host-side launch wrappers for the sm_100a kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rpcb {

// Distance term: l2 squared distance by the Gram trick or directly, or the l1 distance.
enum DistKind { kGaussGram = 0, kGaussDirect = 1, kL1 = 2 };
// Kernel function of the distance term (kernels.hpp:60-79): exp(scale * dd) for Gaussian
// (scale -0.5/sigma^2) and l1 Laplace (scale -1/sigma); Matern 3/2 (scale 1/sigma) and
// Matern 5/2 (scale 1/sigma^2) of the squared l2 distance.
enum KernelFun { kFunExp = 0, kFunMatern32 = 1, kFunMatern52 = 2 };

// Largest block size b (proposals per round) this build accepts; rounds with more than 256
// accepted pivots are appended in groups (api.cu).
constexpr int kMaxBlock = 1024;

// Proposal record layout (one per draw, fp64 words):
//   [0] global id (exact in fp64), [1] ||x||^2, [2, 2+dpad) x, [2+dpad, 2+dpad+ldf) F row
struct RecordLayout {
  int64_t rec;    // record stride (even)
  int64_t xoff;   // = 2
  int64_t foff;   // = 2 + dpad
};

// ---- K2: residual-diagonal scan + inverse-CDF sampling --------------------
// Sequential prefix over all global chunk totals -> chunk_end[], status.
struct ScanStatus {
  double total;       // cumsum[N-1]
  double g2_prev;     // sum over chunks of previous round's ||G||^2 partials
  int32_t exhausted;  // !(total > 0)
  int32_t pad;
};
// Fused chunk prefix (single shard, n_chunks <= kFusedPrefixMax): counter != nullptr makes the
// last CTA of the totals pass run launch_chunk_prefix's serial chain (counter self-resets).
constexpr int kFusedPrefixMax = 1024;
struct FusedPrefix {
  unsigned* counter = nullptr;
  int n_chunks = 0;
  double* chunk_end = nullptr;
  ScanStatus* status = nullptr;
  const double* g2_all = nullptr;
};
// Per-chunk totals of u over this shard's chunks (deterministic tree).
// tile_g2 (optional): the previous update's per-64-row-tile ||G||^2 partials, folded into
// chunk_g2[c] in fixed order (the update kernels' tiles are 64 rows: 64 tiles per chunk).
void launch_chunk_totals(const double* u, int64_t n_loc, int n_chunks, double* totals,
                         cudaStream_t st, const double* tile_g2 = nullptr, int n_tiles = 0,
                         double* chunk_g2 = nullptr, FusedPrefix fp = FusedPrefix(),
                         double* tb = nullptr);
void launch_chunk_prefix(const double* totals_all, const double* g2_all, int n_chunks,
                         double* chunk_end, ScanStatus* status, cudaStream_t st);
// One CTA per draw: draw j uses SplitMix64 counter draw0 + j.
struct SampleParams {
  const double* u;        // this shard's residual diagonal
  const double* X;        // [n_loc][dpad]
  const double* sqn;      // [n_loc]
  const double* F;        // [n_loc][ldf]
  int64_t n_loc, dpad, ldf;
  int64_t n_global;       // N (replay mode searches the global cumsum)
  int kcur;
  int64_t row0;           // global row of local row 0 (multiple of kChunk)
  int chunk0;             // first global chunk of this shard
  int n_chunks_local;
  int n_chunks_global;
  int shard;              // global shard index
  int n_shards;
  const int* shard_chunk0;  // [n_shards + 1] chunk ranges (device)
  const double* chunk_end;  // [n_chunks_global]
  uint64_t seed, draw0;
  int b;
  RecordLayout lay;
  double* records;          // this shard's slot: [b][rec]
  int* owner;               // [b]
  // thread bases of the fast scan, tb[lc][t] = B_(t+1) of local chunk lc (written by the
  // chunk-totals pass or by the fused update); null: the sampler rescans the drawn chunk
  const double* tb = nullptr;
  // with tb: per-chunk totals / ||G||^2 partials of the previous update (fused scan); the
  // sampler then chains the chunk offsets itself (chunk_prefix_kernel's order), writes them
  // to chunk_end and the round status (total, g2_prev, exhausted) to *status (draw 0's CTA)
  const double* totals = nullptr;
  const double* chunk_g2 = nullptr;
  double* chunk_end_out = nullptr;
  ScanStatus* status = nullptr;
};
void launch_sample(const SampleParams& p, cudaStream_t st);
// Replay mode: strictly sequential cumulative_sums (rng.hpp:67-75) over the global
// residual diagonal and std::upper_bound + clamp + plateau walk (rng.hpp:80-96), reference
// rounding; the shard owning the drawn row writes its record.
void launch_replay_scan(const double* u, int64_t n, double* cumsum, ScanStatus* status,
                        cudaStream_t st);
void launch_replay_sample(const SampleParams& p, const double* cumsum, cudaStream_t st);

// ---- K3/K4: H block, rejection sweep, L^{-1} ------------------------------
// part (hblock_scratch_doubles) / tickets (zeroed once, hblock_tickets entries, self-resetting):
// split-K scratch; nullptr = one CTA per tile over the whole k range.
void launch_hblock(const double* prop, RecordLayout lay, int b, int dpad, int d, int kcur,
                   int kind, int kfun, double sigma, double* H, cudaStream_t st,
                   double* part = nullptr, unsigned* tickets = nullptr);
int hblock_splits(int b, int kcur);
// any block of at most b proposals: splits * nb^2 <= max(nb^2, 2 * 296) (hblock_splits)
inline size_t hblock_scratch_doubles(int b) {
  const size_t nb = (size_t)(b + 15) / 16;
  return (nb * nb > 592 ? nb * nb : 592) * 256;
}
inline size_t hblock_tickets(int b) {
  const int nb = (b + 15) / 16;
  return (size_t)nb * nb;
}
struct SweepOut {
  int32_t m;
  int32_t pad;
};
// H: [b][b] row-major (only the lower triangle is read). Outputs pos[m], acc_ids[m],
// lcol[m][b] (column c of the elimination = c-th acceptance), lacc_cm[c][a] (m x m,
// column-major), status.
void launch_sweep(const double* H, int b, uint64_t seed, uint64_t draw0, const double* prop,
                  RecordLayout lay, int* pos, int64_t* acc_ids, double* lcol, double* lacc_cm,
                  SweepOut* out, double* scratch_hp, cudaStream_t st, int accept_all = 0,
                  const ScanStatus* pub_scan = nullptr, char* pub_host = nullptr);
// H[i][i] += shift (block_rpcholesky's LLT retry, rpcholesky.hpp:311-319)
void launch_add_diag(double* H, int b, double shift, cudaStream_t st);
// out[j] = first `words` of record prop[idx[j]] (stride rec), j < m
void launch_gather_records(const double* prop, int64_t rec, int64_t words, const int* idx, int m,
                           double* out, cudaStream_t st);
// The update kernel forms A(R,S) L^{-T} with A(R,S) still in registers when it runs with a
// single warp column (m <= 128): the C-fragment columns a lane holds become its A-operand k
// values, so L^{-1}'s columns are stored in that order inside each 16-column chunk (kslot16).
// Otherwise (m > 128) A(R,S) is parked in F and streamed back from column kcur - koff,
// koff = kcur & 1 (16-byte-aligned TMA boxes), and L^{-1} is stored shifted by koff.
__host__ __device__ inline bool update_regp2(int m) { return m >= 1 && m <= 128; }
// slot of column c inside its 16-column chunk: c % 16 = 8h + 2t + v  ->  4 (2h + v) + t
__host__ __device__ inline int kslot16(int c) {
  return (c & ~15) + 4 * (2 * ((c >> 3) & 1) + (c & 1)) + ((c >> 1) & 3);
}
// column of the [nb][ldl] L^{-1} buffer holding L^{-1}(:, c); perm = 0 forces natural + koff
// (the low-memory path's own use of L^{-1})
__host__ __device__ inline int linv_slot(int c, int m, int koff, int perm) {
  return (perm && update_regp2(m)) ? kslot16(c) : c + koff;
}
// linv_rm[perm_row(a)][linv_slot(c)] = (L^{-1})[a][c], [nb][ldl], zero elsewhere.
void launch_linv(const double* lacc_cm, int m, int nb, int64_t ldl, int koff, double* linv_rm,
                 cudaStream_t st, int perm = 1);
// Same with the accepted count read on the device (*m_dev <= m_max): launched right after
// the sweep, before the host learns m.
void launch_linv_dev(const double* lacc_cm, const int* m_dev, int m_max, int nb, int64_t ldl,
                     int koff, double* linv_rm, cudaStream_t st, int perm = 1);

// ---- residual GEMM on int8 slices (i8gemm.cu) ----------------------------------------
constexpr int kI8Slices = 7;     // base-2^7 digits per operand (Ozaki scheme I)
constexpr int kI8MaxCols = 128;  // output columns (accepted pivots) per launch
constexpr int kI8MinCols = 32;   // fewer accepted pivots: the FP64 DMMA residual is cheaper
// The digits of v (|v| <= 1): V = rint(v 2^48) split into balanced base-2^7 digits, most
// significant first, v = sum_t d_t 2^(-6 - 7 t) + e, |d_t| <= 64, |e| <= 2^-49 (one rounding;
// integer ops only after the first FMA).
__host__ __device__ inline void i8_digits(double v, int (&d)[kI8Slices]) {
  const double t = v * 281474976710656.0 + 6755399441055744.0;  // v 2^48 + 1.5 2^52
  long long V;
#ifdef __CUDA_ARCH__
  V = __double_as_longlong(t) - 0x4338000000000000LL;
#else
  long long bits;
  __builtin_memcpy(&bits, &t, 8);
  V = bits - 0x4338000000000000LL;
#endif
#pragma unroll
  for (int j = kI8Slices - 1; j > 0; --j) {
    const long long dj = ((V + 64) & 127) - 64;
    d[j] = (int)dj;
    V = (V - dj) >> 7;
  }
  d[0] = (int)V;
}
// F(:, c0:c0+nc) -> digit planes [kI8Slices][kcap / 64][plane_rows][64] (int8, kcap % 64 == 0)
void launch_slice_cols(const double* F, int64_t ldf, int64_t n, int c0, int nc, int8_t* planes,
                       int64_t plane_rows, int64_t kcap, cudaStream_t st);
// C(:, :m) = F(:, :kcur) B'^T from F's planes and B' (rows perm_row(a) of bp, as the update's
// B operand), sliced here into bplanes ([kI8Slices][128][kcap] int8) with per-row scales
// (cscale[128]).  C row-major [n_rows][ldc].  Returns 0, or < 0 when not applicable.
int launch_i8_residual(const int8_t* fplanes, int64_t plane_rows, int64_t kcap, int64_t n_rows,
                       const double* bp, int64_t ldbp, int m, int kcur, int8_t* bplanes,
                       double* cscale, double* C, int64_t ldc, cudaStream_t st);

// ---- K5 standalone, Gaussian Gram, d <= 32: Gram on tcgen05 int8 digit planes (i8cols.cu) ----
constexpr int kI8ColsMaxD = 32;
constexpr int kI8ColsSlices = 8;  // digits per point coordinate (i8cols.cu)
// launches with fewer columns stay on the FP64 kernel (C4 points: i8 slower at m <= 40,
// faster from m = 48: 217k vs 167k columns/s)
constexpr int kI8ColsMinM = 48;
// bytes of the point digit planes ([kI8ColsSlices][round_up(n, 128)][32] int8)
int64_t i8cols_plane_bytes(int64_t n);
// planes + per-row exponents (int[n]) of the packed points X [n][dpad]
void launch_i8cols_prep(const double* X, int64_t dpad, int d, int64_t n, int8_t* planes,
                        int* xexp, cudaStream_t st);
// out[c ld_out + r] = k(x_r, x_{id_c}) for c < m <= 128 (ids in the proposal records' slot 0);
// bplanes: kI8ColsSlices * 128 * 32 bytes, cinfo: 384 doubles (scratch).  0, or < 0 on failure.
int launch_i8cols(const int8_t* planes, const int* xexp, const double* sqn, int64_t n,
                  const double* prop, int64_t rec, int m, int kfun, double escale,
                  int8_t* bplanes, double* cinfo, double* out, int64_t ld_out, cudaStream_t st);

// ---- K5+K6: fused kernel columns + residual GEMM + L^{-T} + diag update ----
struct UpdateParams {
  const double* X; int64_t dpad; int dchunks;   // X shard [n_loc][dpad]
  int d;                                        // true dimension (distance loops skip the padding)
  const double* sqn;                            // ||x||^2 [n_loc]
  double* F; int64_t ldf; int kcur;             // F shard [n_loc][ldf]
  double* u;                                    // residual diagonal [n_loc]
  int64_t n_loc; int64_t row0;
  const double* xs; const double* fs; int64_t ldfs;  // accepted operands [256][dpad|ldfs], rows perm_row(n)
  const double* sqnS; const double* idS;        // [256] logical column order
  int m;
  const double* linv; int64_t ldl;             // L^{-1} rows perm_row(a), [256][ldl]
  double sigma; int kind;
  double escale;            // kernel-function scale (KernelFun), host-computed
  int kfun;                 // KernelFun
  double* tile_g2;                              // [n_tiles] per-CTA ||G||^2 partial (row order)
  int g2_accum;                                 // add to tile_g2 instead of storing (grouped rounds)
  // columns-only mode (standalone K5: A(:, S) -> cols_out col-major [m][ld_out])
  int columns_only; double* cols_out; int64_t ld_out;
  // Scan partials (single warp column, 64-row tiles, tsum != null): the epilogue also writes
  // each 16-row run's sequential sum of the new u (tsum[row / 16] = chunk_scan_core's
  // per-thread sum), so the next round's scan reads 1/16 of u (launch_chunk_chain).
  double* tsum;
  // Residual GEMM precomputed on the tensor cores (launch_i8_residual; m <= 128): the kernel
  // skips its own F B'^T phase and adds cext[row][col] (row-major, ld ldce) instead.
  const double* cext; int64_t ldce;
  // RPC_DEBUG_TIMING: per-CTA cycle counters per phase ([grid][8] u64), or null
  unsigned long long* phase_clk;
  // RPC_DEBUG_TRACE: CTA 0 per-group phase clocks [G][64 tiles][8] (debug only)
  unsigned long long* trace;
};
// Row-tile height used for m accepted columns (128 or 64), or -1 if m unsupported.
int update_tile_rows(int m);
// Launch; returns the tile height, or < 0 on failure (-1 unsupported m, -2 smem attr, -3 TMA map).
int launch_update(const UpdateParams& p, cudaStream_t st);
// B'[perm_row(n)][k] = -(L^{-1} F_S)[n][k] for k < kcur (the residual GEMM's B operand with
// the triangular solve folded in); linv_rm as written by launch_linv*, F_S rows from the
// proposal records of the accepted positions.  *m_dev = accepted count (<= m_max).
// m_dev == nullptr: m = m_max.  Grouped rounds (lext != nullptr): F_S columns
// [kprop, kcur) are L(g0 + a, k - kprop), read from the sweep's column-major m_full x m_full L.
void launch_bprime(const double* linv_rm, int64_t ldl, int koff, const double* prop,
                   RecordLayout lay, const int* pos, const int* m_dev, int m_max, int kcur,
                   double* bp, int64_t ldbp, cudaStream_t st, const double* lext = nullptr,
                   int m_full = 0, int g0 = 0, int kprop = -1);
// linv (as launch_linv_dev, update layout) + B' = -L^{-1} F_S (forward substitution, into
// bp rows perm_row(a) < m, columns < kcur) + the accepted X rows / norms / ids (as
// launch_gather_accepted without F rows; n_rows operand rows, zero beyond m), one launch.
// Sweep + round prep in one cooperative launch (b <= 128): CTA 0 sweeps (as launch_sweep
// with the mapped-memory publish, plus a sequence word SweepOut::pad = epoch written last),
// the other CTAs form L^{-1}, B' and the accepted operands (as launch_round_prep with
// m_dev) behind it from its per-block progress word.  prog: one u64 (any initial value);
// aidx: [b] ints.  epoch must differ between launches sharing prog.  Returns the grid size,
// or < 0 when the launch is not possible (caller falls back to the two launches).
int launch_sweep_prep(const double* H, int b, uint64_t seed, uint64_t draw0, const double* prop,
                      RecordLayout lay, int* pos, int64_t* acc_ids, double* lcol,
                      double* lacc_cm, SweepOut* out, const ScanStatus* pub_scan,
                      char* pub_host, unsigned long long* prog, int* aidx, unsigned epoch,
                      int nb, int64_t ldl, double* linv_rm, int kcur, double* bp, int64_t ldbp,
                      int dpad, double* xs, double* sqnS, double* idS, double xscale,
                      int n_rows, cudaStream_t st);
void launch_round_prep(const double* lacc_cm, int m_host, const int* m_dev, int m_max, int nb,
                       int64_t ldl, int koff, double* linv_rm, const double* prop,
                       RecordLayout lay, const int* pos, int kcur, double* bp, int64_t ldbp,
                       int dpad, double* xs, double* sqnS, double* idS, double xscale,
                       int n_rows, cudaStream_t st);
// Gathers the accepted pivots' X rows, F rows (first kcur columns), norms and ids from the
// proposal records into the update kernel's operand buffers (rows at perm_row(n), n < nb).
// X rows are multiplied by xscale: the Gram kernel passes -2 (gram_xscale), so the DMMA
// product is -2 X(R,:) X(S,:)^T bit for bit (a power-of-two scale is exact).
void launch_gather_accepted(const double* prop, RecordLayout lay, const int* pos, int m, int nb,
                            int kcur, int dpad, double* xs, double* fs, int64_t ldfs,
                            double* sqnS, double* idS, cudaStream_t st,
                            const int* m_dev = nullptr, double xscale = 1.0);
inline double gram_xscale(int kind) { return kind == kGaussGram ? -2.0 : 1.0; }
// From the update's 16-row run sums (UpdateParams::tsum) and tile ||G||^2 partials: per
// local chunk the thread bases tb[c][t] = B_(t+1), totals[c] and chunk_g2[c] (tile order),
// with chunk_totals_kernel's serial association (bitwise the same values).
void launch_chunk_chain(const double* tsum, const double* tile_g2, int64_t n_loc, int n_chunks,
                        double* tb, double* totals, double* chunk_g2, cudaStream_t st);
// per-chunk sum of per-tile partials (tile = rows_per_tile rows)
void launch_tile_to_chunk(const double* tile_g2, int n_tiles, int tiles_per_chunk,
                          int n_chunks_local, double* chunk_g2, cudaStream_t st);
// per-chunk ||F(rows, :k)||^2
void launch_fsq_chunks(const double* F, int64_t ldf, int64_t n_loc, int k, int n_chunks_local,
                       double* chunk_out, cudaStream_t st);
// F row-major [n_loc][ldf] columns [c0, c0+nc) -> out col-major [nc][ld_out]
void launch_f_to_colmajor(const double* F, int64_t ldf, int64_t n_loc, int c0, int nc,
                          double* out, int64_t ld_out, cudaStream_t st);
// ---- low-memory variant (accelerated_rpcholesky_lowmem, rpcholesky.hpp:408-485) ----
// State: pivot records piv[k][prec] (id, ||x||^2, x), Linv = L^{-1} of the pivot block
// ([cap][ldw] row-major, lower), L ([cap][ldw] row-major, lower), u.  No N x k factor.
// Per round the diagonal update is  u -= rowsq(A(R, S_all) W^T),  W = rows
// [kold, kold+m) of the new L^{-1}: the kernel block A(R, S_all) is regenerated tile
// by tile in shared memory and never leaves the SM (lowmem.cu).
struct LowmemParams {
  const double* X; int64_t dpad; int dchunks; int d;  // X shard [n_loc][dpad]
  const double* sqn;                                  // ||x||^2 [n_loc]
  double* u;                                          // residual diagonal [n_loc]
  int64_t n_loc; int64_t row0;
  const double* piv; int64_t prec;                    // pivot records [knew][prec]
  const double* W; int64_t ldw;                       // W = Linv + kold * ldw, [m][knew]
  int m, kold, knew;
  int kind; double escale; int kfun;                  // DistKind, KernelFun scale, KernelFun
  double* tile_g2;                                    // [n_tiles] per-tile ||G||^2
  // product mode (kernel_matvec / predict, krr.hpp:143-162, 227-250): instead of the
  // diagonal update, out[row * ld_out + j] = (A(R, S) W^T)[row][j] + add_coef * add_vec[row]
  // + add_const for j < m.  pin = 0 disables the same-index distance pin (cross blocks
  // between different point sets, oracle.hpp:149-166).
  int out_mode; double* out; int64_t ld_out;
  const double* add_vec; double add_coef; double add_const;
  int pin;
};
// Returns the tile height (64), or < 0 on failure (-1 unsupported m/d, -2 attr, -3 map).
int launch_lowmem(const LowmemParams& p, cudaStream_t st);
// C[M x N] = alpha op(A) op(B) + beta C, row-major fp64 (op = transpose when t* != 0).
void launch_gemm(int M, int N, int K, double alpha, const double* A, int64_t lda, int ta,
                 const double* B, int64_t ldb, int tb, double beta, double* C, int64_t ldc,
                 cudaStream_t st);
// K[j][i] = A(prop_j, piv_i) for j < b, i < k (kentry.cuh).
void launch_kprop(const double* prop, RecordLayout lay, int b, const double* piv, int64_t prec,
                  int k, int d, int kind, int kfun, double sigma, double* K, int64_t ldk,
                  cudaStream_t st);
// Appends the m accepted pivots: piv rows, F_S = prop F rows -> fs[m][ldk] and L rows
// [kold+a] = (F_S[a], L_sel[a]), Linv rows [kold+a][kold..] = L_sel^{-1}[a] (from linv_rm,
// rows perm_row(a), koff 0).
void launch_lowmem_append(const double* prop, RecordLayout lay, const int* pos, int m, int kold,
                          int64_t prec, const double* lacc_cm, const double* linv_rm, int64_t ldl,
                          double* piv, double* fs, int64_t ldk, double* Lrm, double* Linv,
                          int64_t ldw, cudaStream_t st);
// chol (k x k column-major, lower) from the row-major L.
void launch_lowmem_chol(const double* Lrm, int64_t ldw, int k, double* chol, cudaStream_t st);

// ---- symmetric kernel matvec (krr.hpp:143-162, one right-hand side), symv.cu ----------------
// out = A v + add_coef * add_vec + add_const over the training points themselves, each
// 1024 x 1024 block of the lower block triangle generated once and used for both A v and
// A^T v; deterministic.  v: [n] (16-byte aligned, row stride ldv for the TMA map).
int64_t symv_scratch_doubles(int64_t n);
bool launch_symv(const double* X, int64_t dpad, int d, const double* sqn, const double* rec,
                 int64_t prec, const double* v, int64_t ldv, int64_t n, int kind, int kfun,
                 double escale, double* scratch, const double* add_vec, double add_coef,
                 double add_const, double* out, cudaStream_t st);

// ---- KRR preconditioner core (krr.hpp:30-70), krr_core.cu: row-major [kc][kc] ----------
// kc = k rounded up to 64; entries beyond k hold the identity.  Lower triangle only.
int64_t core_dim(int k);
size_t core_syrk_scratch_doubles(int k);
// core = F^T F + mu I  (F row-major [n][ldf], first k columns; DMMA, deterministic)
void launch_core_syrk(const double* F, int64_t ldf, int64_t n, int k, double mu, double* core,
                      double* scratch, cudaStream_t st);
// core <- L (Cholesky, lower); *info = 1 + first failing column block start (caller zeroes it)
void launch_core_potrf(double* core, int64_t kc, int* info, cudaStream_t st);
// t <- (L L^T)^{-1} t   (t: kc doubles, zero beyond k)
void launch_core_potrs(const double* L, int64_t kc, double* t, cudaStream_t st);

// X (host layout already on device as col-major or row-major) -> padded row-major + norms
// *nonfinite is set to 1 if any input coordinate is NaN/Inf (DataMatrix, data_matrix.hpp:26-28)
void launch_pack_points(const double* src, int64_t n_loc, int d, int64_t ld_src,
                        int src_row_major, int64_t dpad, double* X, double* sqn,
                        int* nonfinite, cudaStream_t st);
void launch_fill(double* p, int64_t n, double v, cudaStream_t st);

}  // namespace rpcb
