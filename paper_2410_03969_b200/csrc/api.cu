// api.cu — host runtime and C-ABI of librpchol_b200.so.
//
// Replaces rpchol::accelerated_rpcholesky (rpcholesky.hpp:338-401) for kernel
// oracles (oracle.hpp:243-327).  The host drives the round loop; all N-sized
// work stays on the device(s).  One host<->device synchronisation per round
// reads back the round's status words (scan total, accepted count, pivot ids)
// that the reference's PivotTrace needs anyway.
//
// Row sharding: global scan chunks of 4096 rows are split into
// P equal contiguous chunk ranges, one per shard.  A shard is either this
// process's GPU (NCCL mode, one process per GPU) or one of several virtual
// shards on a single GPU (collectives become local device copies).  Per round
// the shards exchange only: chunk totals (+ previous round ||G||^2 partials),
// and the b proposal records (id, ||x||^2, x, F row).  The sweep and L^{-1}
// are computed redundantly and bit-identically on every shard.
#include <atomic>
#include <memory>

#include "runtime.h"

namespace rpcb_rt {

__global__ void chol_gather_kernel(const double* __restrict__ F, int64_t ldf, int64_t row0,
                                   int64_t n_loc, const int64_t* __restrict__ piv, int64_t k,
                                   double* __restrict__ out_rm) {
  const int64_t i = blockIdx.x;
  const int64_t lr = piv[i] - row0;
  if (lr < 0 || lr >= n_loc) return;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) out_rm[j * k + i] = F[lr * ldf + j];
}

// First factor width at which a round's residual GEMM goes to the tensor cores (i8gemm.cu):
// below it the FP64 DMMA phase of the update is as fast (C4, two-pass kernel: 33.0 / 32.9 / 33.4 ms
// at 192 / 256 / 384).
static int64_t i8_min_k_env() {
  const char* e = std::getenv("RPC_I8_MIN_K");
  return e ? std::atoll(e) : 256;
}

// Launch tags of the fused sweep + prep (its progress word and the host sequence word):
// unique per launch within the process.
static unsigned next_epoch() {
  static std::atomic<unsigned> e{0x5eed0001u};
  unsigned v = e.fetch_add(1u);
  return v ? v : e.fetch_add(1u);
}

// Host wait for the fused launch's status publish: spin on the sequence word the sweep
// writes last into mapped pinned memory (no event-completion round trip).  Every few
// thousand polls the launch's event is queried: an event that completed (or failed) without
// the word means a fault, reported instead of spinning forever.
static void wait_published(const int32_t* seq, unsigned epoch, cudaEvent_t ev) {
  const volatile int32_t* w = seq;
  for (unsigned it = 1;; ++it) {
    if ((unsigned)*w == epoch) break;
    if ((it & 4095u) == 0) {
      const cudaError_t e = cudaEventQuery(ev);
      if (e == cudaErrorNotReady) continue;
      if ((unsigned)*w == epoch) break;
      CK(e);
      CK(cudaGetLastError());
      throw RpcError{RPC_ECUDA, "round status was not published by the sweep"};
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// The factorization proper.  `src` points to this process's shard rows (device
// memory when src_on_device, else host memory of the full X).
//
// lowmem: accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485) — the same proposals,
// sweep and stopping rules, but no N x k factor: the proposals' factor rows come from
// A(S', S) L^{-T}, and the diagonal update regenerates A(R, S_all) inside the update
// kernel (lowmem_impl.cuh).  State: X, u, pivot records, L and L^{-1} (k x k).
// RPC_DEBUG_TRACE: print CTA 0's per-group, per-tile phase clocks of each update launch
static void dump_trace(const DBuf& buf, int m, int64_t kcur, cudaStream_t st) {
  std::vector<unsigned long long> h(buf.bytes / 8);
  CK(cudaMemcpyAsync(h.data(), buf.p, buf.bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::fprintf(stderr, "[trace] m=%d kcur=%lld\n", m, (long long)kcur);
  for (int g = 0; g < 2; ++g)
    for (int t = 0; t < 64; ++t) {
      const unsigned long long* r = &h[(g * 64 + t) * 8];
      if (!r[0]) continue;
      std::fprintf(stderr, "[trace] %d %d %llu %llu %llu %llu %llu %llu %llu\n", g, t, r[0], r[1], r[2],
                   r[3], r[4], r[5], r[6]);
    }
}

void run_factorization(rpc_ctx* ctx, const double* src, bool src_on_device, int64_t n,
                       int64_t d, int64_t ldx, int layout, const rpc_kernel_spec& kspec,
                       rpc_run_config cfg, rpc_result* res, bool lowmem, int algo,
                       HostSink sink) {
  int kind = 0;
  validate(n, d, kspec, cfg, kind);
  double kscale = 0.0;
  const int kfun = kernel_fun(kspec, &kscale);
  if (algo != kAlgoAccelerated && lowmem) raise(RPC_EINVAL, "low-memory mode is accelerated-only");
  if (sink.p && lowmem) raise(RPC_EINVAL, "low-memory result has no factor to stream");
  if (lowmem && round_up(d, 16) > 128)
    raise(RPC_EINVAL, "accelerated_rpcholesky_lowmem: this build supports d <= 128");
  if (lowmem && cfg.block_size > 256)
    raise(RPC_EINVAL, "accelerated_rpcholesky_lowmem: this build supports block size <= 256");
  if (layout != RPC_COL_MAJOR && layout != RPC_ROW_MAJOR) raise(RPC_EINVAL, "unknown layout");
  const bool replay = (cfg.flags & RPC_FLAG_REPLAY_SCAN) != 0;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int b = (int)cfg.block_size;
  int64_t cap = cfg.mode == RPC_FIXED_ROUNDS ? cfg.rounds * cfg.block_size
                                             : cfg.target_rank + cfg.block_size;
  cap = std::min(cap, n);
  const int64_t ldf = round_up(std::max<int64_t>(cap, 1), 16);
  const int64_t dpad = round_up(d, 16);
  const Layout L = make_layout(n, ctx->nshards());
  RecordLayout lay;
  lay.xoff = 2;
  lay.foff = 2 + dpad;
  lay.rec = 2 + dpad + ldf;

  NvtxRange nv_all(lowmem ? "rpc:accelerated_rpcholesky_lowmem"
                           : algo == kAlgoBlock  ? "rpc:block_rpcholesky"
                           : algo == kAlgoSimple ? "rpc:simple_rpcholesky"
                                                 : "rpc:accelerated_rpcholesky");
  using clk = std::chrono::steady_clock;
  const auto h0 = clk::now();
  auto ms_since = [](clk::time_point a) {
    return std::chrono::duration<double, std::milli>(clk::now() - a).count();
  };
  res->ctx = ctx;
  res->n = n;
  res->d = d;
  res->ldf = ldf;
  res->b = b;
  res->lowmem = lowmem;
  rpc_timing& tm = res->timing;
  int64_t launches = 0;

  // ---- per-shard state + upload -------------------------------------------
  Ev ev_up0, ev_up1, ev_t0, ev_t1;
  CK(cudaEventRecord(ev_up0.e, st));
  res->shards.resize(ctx->nvirt);
  DBuf nonfinite(ctx, sizeof(uint64_t));  // int flag in a zeroed 64-bit word (owner reduce)
  CK(cudaMemsetAsync(nonfinite.p, 0, sizeof(uint64_t), st));
  int64_t max_tiles = 0;
  for (int v = 0; v < ctx->nvirt; ++v) {
    Shard& s = res->shards[v];
    s.gidx = ctx->first_shard() + v;
    s.row0 = L.row0(s.gidx);
    s.n_loc = L.rows(s.gidx);
    s.chunk0 = s.gidx * L.cpr;
    s.nchunks = L.chunks(s.gidx);
    const int64_t nl = std::max<int64_t>(s.n_loc, 1);
    s.X = DBuf(ctx, sizeof(double) * nl * dpad);
    s.sqn = DBuf(ctx, sizeof(double) * nl);
    if (!lowmem) s.F = DBuf(ctx, sizeof(double) * nl * ldf);
    s.u = DBuf(ctx, sizeof(double) * nl);
    s.tile_g2 = DBuf(ctx, sizeof(double) * (nl / 64 + 2));
    max_tiles = std::max<int64_t>(max_tiles, nl / 64 + 2);
    if (s.n_loc == 0) continue;
    // stage this shard's raw rows on the device, then pack (pad, norms)
    const double* dsrc = nullptr;
    DBuf tmp;
    int64_t ld_src = 0;
    if (src_on_device) {
      // x_dev holds this process's rows; with virtual shards that is all rows
      const int64_t off = ctx->nvirt > 1 ? s.row0 : 0;
      dsrc = layout == RPC_ROW_MAJOR ? src + off * ldx : src + off;
      ld_src = ldx;
    } else {
      if (layout == RPC_ROW_MAJOR) {
        tmp = DBuf(ctx, sizeof(double) * s.n_loc * d);
        if (ldx == d)  // contiguous rows: one linear copy (a pitched copy of 8d-byte rows is slow)
          CK(cudaMemcpyAsync(tmp.p, src + s.row0 * ldx, sizeof(double) * s.n_loc * d,
                             cudaMemcpyHostToDevice, st));
        else
          CK(cudaMemcpy2DAsync(tmp.p, d * sizeof(double), src + s.row0 * ldx, ldx * sizeof(double),
                               d * sizeof(double), s.n_loc, cudaMemcpyHostToDevice, st));
        ld_src = d;
      } else {
        tmp = DBuf(ctx, sizeof(double) * s.n_loc * d);
        CK(cudaMemcpy2DAsync(tmp.p, s.n_loc * sizeof(double), src + s.row0, ldx * sizeof(double),
                             s.n_loc * sizeof(double), d, cudaMemcpyHostToDevice, st));
        ld_src = s.n_loc;
      }
      dsrc = tmp.as<double>();
    }
    launch_pack_points(dsrc, s.n_loc, (int)d, ld_src, layout == RPC_ROW_MAJOR, dpad,
                       s.X.as<double>(), s.sqn.as<double>(), nonfinite.as<int>(), st);
    CK(cudaGetLastError());
    launch_fill(s.u.as<double>(), s.n_loc, 1.0, st);  // u = max(diag, 0) = 1 (oracle.hpp:263)
    launches += 2;
    if (tmp.p) CK(cudaStreamSynchronize(st));  // tmp returns to the pool
  }
  CK(cudaEventRecord(ev_up1.e, st));
  {  // DataMatrix rejects non-finite entries (data_matrix.hpp:26-28); every rank agrees
    allreduce_owner(ctx, nonfinite.p, 1);
    uint64_t bad = 0;
    CK(cudaMemcpyAsync(&bad, nonfinite.p, sizeof bad, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad) raise(RPC_EINVAL, "DataMatrix: non-finite entry");
  }

  // ---- replicated per-round buffers ---------------------------------------
  const int P = L.P;
  DBuf totals_all(ctx, sizeof(double) * L.ncg), g2_all(ctx, sizeof(double) * L.ncg),
      chunk_end(ctx, sizeof(double) * L.ncg);
  // proposal records: every draw's owner writes its slot; across processes the slots are
  // combined by the owner reduce (zeroed first), so each GPU receives b records, not P b
  DBuf prop(ctx, sizeof(double) * b * lay.rec);
  DBuf owner(ctx, sizeof(int) * b), Hbuf(ctx, sizeof(double) * b * b),
      lcol(ctx, sizeof(double) * b * b), lacc(ctx, sizeof(double) * b * b);
  const int64_t ldl = 272, nbl = 256;  // L^{-1} columns shifted by kcur & 1 (update.cu)
  DBuf linv(ctx, sizeof(double) * nbl * ldl), pos(ctx, sizeof(int) * b),
      acc_ids(ctx, sizeof(int64_t) * b), hp(ctx, sizeof(double) * ((size_t)b * (b + 1) / 2 + 1));
  DBuf status(ctx, sizeof(ScanStatus) + sizeof(SweepOut));
  // split-K H block scratch
  DBuf hb_part(ctx, sizeof(double) * hblock_scratch_doubles(b)),
      hb_tick(ctx, sizeof(unsigned) * hblock_tickets(b));
  CK(cudaMemsetAsync(hb_tick.p, 0, hb_tick.bytes, st));
  // accepted-pivot operands of the fused update (rows permuted, see common.cuh perm_row)
  DBuf xs(ctx, sizeof(double) * 256 * dpad), fs(ctx, sizeof(double) * 256 * ldf),
      sqnS(ctx, sizeof(double) * 256), idS(ctx, sizeof(double) * 256);
  DBuf shard_c0(ctx, sizeof(int) * (P + 1));
  // Blocks beyond 128 proposals: a round's accepted set is appended in balanced groups of at
  // most kGroup pivots (block Cholesky: group g is eliminated against F extended by the
  // earlier groups' columns, whose rows at S_g are L(S_g, S_<g) from the sweep), each group
  // one update launch of the single-warp-column kernel (A(R,S) L^{-T} from registers); L_gg
  // is copied out of the sweep's L for its inverse.  Against one two-warp-column launch for
  // 128 < m <= 256 (A parked in F): C5 1234 -> 1171 ms, same flops.
  constexpr int kGroup = 128;
  const bool grouped = b > kGroup && !lowmem;
  DBuf lsub;
  if (grouped) lsub = DBuf(ctx, sizeof(double) * kGroup * kGroup);
  DBuf prefix_counter(ctx, sizeof(unsigned));
  CK(cudaMemsetAsync(prefix_counter.p, 0, sizeof(unsigned), st));
  // fast-scan thread bases (sampler) and the update-fused scan's chunk bookkeeping
  DBuf tb_all(ctx, sizeof(double) * (size_t)L.ncg * kScanThreads);
  const bool fuse_scan_ok = !lowmem && !replay && L.ncg <= 4096 &&
                            std::getenv("RPC_NO_FUSED_SCAN") == nullptr;
  std::vector<DBuf> scan_tsum(res->shards.size());  // per shard: 16-row run sums of u
  if (fuse_scan_ok)
    for (size_t si = 0; si < res->shards.size(); ++si) {
      const int64_t ntiles64 = (res->shards[si].n_loc + 63) / 64;
      scan_tsum[si] = DBuf(ctx, sizeof(double) * (size_t)std::max<int64_t>(1, 4 * ntiles64));
    }
  // Residual GEMM on the tensor cores (i8gemm.cu): F's int8 digit planes are kept beside F
  // (each round appends its columns), and rounds with kcur >= RPC_I8_MIN_K (default 256) and
  // m <= 128 compute F B'^T there; the update kernel then adds it.  Used when the planes fit
  // next to F (7 bytes per factor entry); RPC_NO_I8 forces the FP64 DMMA path.
  // (block_rpcholesky too: same update path, |F| <= 1 holds with the diagonal shift; not
  // simple_rpcholesky: one column per round)
  bool i8_ok = !lowmem && (algo == kAlgoAccelerated || algo == kAlgoBlock) &&
               cap > i8_min_k_env() &&
               !(cfg.flags & RPC_FLAG_FP64_RESIDUAL) && std::getenv("RPC_NO_I8") == nullptr;

  const int64_t i8_min_k = i8_min_k_env();
  const int64_t i8_kcap = round_up(std::max<int64_t>(cap, 1), 64);
  std::vector<DBuf> i8_planes(res->shards.size());
  std::vector<int64_t> i8_rows(res->shards.size(), 0);
  DBuf i8_bplanes, i8_cscale, i8_c;
  if (i8_ok) {
    // (the planes take 7 bytes per factor entry: when they do not fit next to F the run
    // stays on the FP64 DMMA path instead of failing)
    try {
      int64_t maxrows = 0;
      for (size_t si = 0; si < res->shards.size(); ++si) {
        i8_rows[si] = round_up(std::max<int64_t>(res->shards[si].n_loc, 1), 128);
        maxrows = std::max(maxrows, i8_rows[si]);
        i8_planes[si] = DBuf(ctx, (size_t)kI8Slices * i8_rows[si] * i8_kcap);
      }
      i8_bplanes = DBuf(ctx, (size_t)kI8Slices * kI8MaxCols * i8_kcap);
      i8_cscale = DBuf(ctx, sizeof(double) * kI8MaxCols);
      i8_c = DBuf(ctx, sizeof(double) * (size_t)maxrows * kI8MaxCols);
    } catch (const RpcError&) {
      cudaGetLastError();
      for (auto& b : i8_planes) b.release();
      i8_bplanes.release();
      i8_cscale.release();
      i8_c.release();
      i8_ok = false;
    }
  }
  int64_t i8_launches = 0;
  double tc_ops = 0.0, tc_fl = 0.0;
  std::vector<Ev> tc_ev, sl_ev;  // (start, end) pairs: tensor-core residual, plane appends
  // true while the last update's 16-row run sums (tsum) describe the current u: the next
  // scan then chains them (launch_chunk_chain, 1/16 of u's bytes) instead of a totals pass
  // over u, and the sampler chains the chunk offsets
  bool scan_fresh = false;
  // fused sweep + round prep (accelerated, b <= 128, one group): progress word + acceptance map
  DBuf sweep_prog(ctx, sizeof(unsigned long long)), sweep_aidx(ctx, sizeof(int) * b);
  CK(cudaMemsetAsync(sweep_prog.p, 0, sizeof(unsigned long long), st));
  const bool fused_prep_ok = std::getenv("RPC_NO_FUSED_PREP") == nullptr;
  DBuf kept_idx, propk;  // block / simple: kept proposals (first draw of each distinct id)
  if (algo != kAlgoAccelerated) {
    kept_idx = DBuf(ctx, sizeof(int) * b);
    propk = DBuf(ctx, sizeof(double) * b * lay.rec);
  }
  DBuf cumsum, u_all;
  if (replay) cumsum = DBuf(ctx, sizeof(double) * n);
  // replay with several shards: the sequential scan needs the whole residual diagonal, so
  // every shard gathers it (global row order = shard slot order) and scans it identically
  if (replay && P > 1) u_all = DBuf(ctx, sizeof(double) * (size_t)L.ncg * kChunk);
  // low-memory state (replicated): pivot records, L and L^{-1} row-major [cap][ldf],
  // per-round scratch K(S', S), F_S and F_S L^{-1}
  const int64_t prec = 2 + dpad;
  DBuf piv, Lrm, Linv, Kp, fsl, T1;
  if (lowmem) {
    piv = DBuf(ctx, sizeof(double) * cap * prec);
    Lrm = DBuf(ctx, sizeof(double) * cap * ldf);
    Linv = DBuf(ctx, sizeof(double) * cap * ldf);
    Kp = DBuf(ctx, sizeof(double) * b * ldf);
    fsl = DBuf(ctx, sizeof(double) * b * ldf);
    T1 = DBuf(ctx, sizeof(double) * b * ldf);
    CK(cudaMemsetAsync(Lrm.p, 0, Lrm.bytes, st));
    CK(cudaMemsetAsync(Linv.p, 0, Linv.bytes, st));
  }
  {
    std::vector<int> c0(P + 1);
    for (int s = 0; s <= P; ++s) c0[s] = s * L.cpr;
    CK(cudaMemcpyAsync(shard_c0.p, c0.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(totals_all.p, 0, sizeof(double) * L.ncg, st));
  CK(cudaMemsetAsync(g2_all.p, 0, sizeof(double) * L.ncg, st));
  ScanStatus* d_scan = status.as<ScanStatus>();
  SweepOut* d_sweep = reinterpret_cast<SweepOut*>(d_scan + 1);

  // pinned host mirror: ScanStatus | SweepOut | proposal ids (double) [b] | accepted ids [b]
  const size_t hbytes = sizeof(ScanStatus) + sizeof(SweepOut) + sizeof(double) * b +
                        sizeof(int64_t) * b + 64;
  char* hbuf = static_cast<char*>(ctx->pinned(hbytes));
  ScanStatus* h_scan = reinterpret_cast<ScanStatus*>(hbuf);
  SweepOut* h_sweep = reinterpret_cast<SweepOut*>(h_scan + 1);
  double* h_prop_ids = reinterpret_cast<double*>(h_sweep + 1);
  int64_t* h_acc_ids = reinterpret_cast<int64_t*>(h_prop_ids + b);
  Ev ev_pub;                  // status published (mapped-memory path)
  char* hbuf_dev = nullptr;  // device alias of the pinned status buffer (UVA mapping)
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&hbuf_dev), hbuf, 0) != cudaSuccess) {
    cudaGetLastError();
    hbuf_dev = nullptr;
  }

  const double trace_a = (double)n;  // sum of diag(A) = N exactly
  int64_t kcur = 0;
  double captured_sq = 0.0;
  bool pending_g2 = false;
  std::vector<Ev> upd_ev;
  upd_ev.reserve(8);
  std::vector<std::pair<int, int64_t>> upd_info;
  const bool dbg_phase = std::getenv("RPC_DEBUG_PHASES") != nullptr;
  const bool dbg_trace = std::getenv("RPC_DEBUG_TRACE") != nullptr;
  const bool dbg_gaps = std::getenv("RPC_DEBUG_GAPS") != nullptr;
  std::vector<Ev> gap_ev;
  gap_ev.reserve(64);
  // RPC_DEBUG_CHAIN: an event after every per-round stage; the elapsed time between
  // consecutive marks is charged to the later label (device timeline incl. launch gaps)
  const bool dbg_chain = std::getenv("RPC_DEBUG_CHAIN") != nullptr;
  std::vector<std::pair<const char*, Ev>> chain_ev;
  chain_ev.reserve(dbg_chain ? 1024 : 0);
  double host_pre_us = 0.0, host_launch_us = 0.0;  // RPC_DEBUG_CHAIN: wake -> launch, launch call
  auto cmark = [&](const char* what) {
    if (!dbg_chain) return;
    chain_ev.emplace_back(what, Ev());
    CK(cudaEventRecord(chain_ev.back().second.e, st));
  };
  DBuf trace_buf(ctx, dbg_trace ? sizeof(unsigned long long) * 2 * 64 * 8 : 8);
  DBuf phase_clk(ctx, dbg_phase ? sizeof(unsigned long long) * 8 * 4096 : 8);
  std::vector<double> upd_flops;
  double update_ms = 0.0, flops = 0.0, bytes = 0.0;
  int64_t upd_launches = 0;

  // Factor streaming (HostSink): round r's finished columns F(:, kcur:kcur+m) are final, so
  // a second stream transposes them to column-major and copies them to the host while the
  // next rounds compute (double-buffered staging, one half per round in flight).
  cudaStream_t cst = ctx->copy_stream;
  int64_t rows_here = 0;
  for (const Shard& s : res->shards) rows_here += s.n_loc;
  DBuf sink_tmp[2];
  std::vector<Ev> sink_ev(sink.p ? 2 : 0);
  int sink_slot = 0;
  if (sink.p) {
    if (sink.cols < cap || sink.ld < rows_here)
      raise(RPC_EINVAL, "factor buffer too small (needs this process's rows x min(N, k + b))");
    sink_tmp[0] = DBuf(ctx, sizeof(double) * std::max<int64_t>(rows_here, 1) * b);
    sink_tmp[1] = DBuf(ctx, sizeof(double) * std::max<int64_t>(rows_here, 1) * b);
  }
  // On every exit path (an exception mid-loop included) wait for the factor copies still
  // queued on the copy stream before the staging halves, F (via the result) and the
  // caller's registered buffer can be released or reused.
  struct CopyDrain {
    cudaStream_t s;
    ~CopyDrain() {
      if (s) cudaStreamSynchronize(s);
    }
  } copy_drain{sink.p ? cst : nullptr};
  // Digit-plane appends run on a third stream: a round's append is only read by the next
  // tensor-core product, so it overlaps the next round's chain (scan, sampler, H block, sweep,
  // prep: single-CTA kernels that leave the GPU idle) instead of preceding it.  RPC_NO_AUX_SLICE
  // keeps it on the main stream.
  static const bool aux_slice = std::getenv("RPC_NO_AUX_SLICE") == nullptr;
  cudaStream_t ast = (i8_ok && aux_slice && ctx->aux_stream) ? ctx->aux_stream : st;
  Ev ev_upd_done, ev_slice_done;
  bool slice_pending = false;
  CopyDrain aux_drain{ast != st ? ast : nullptr};
  const double setup_ms = ms_since(h0);
  const auto h1 = clk::now();
  CK(cudaEventRecord(ev_t0.e, st));
  for (int64_t round = 0;; ++round) {
    if (cfg.mode == RPC_FIXED_ROUNDS ? round >= cfg.rounds : kcur >= cfg.target_rank) break;
    NvtxRange nv_round("rpc:round");
    cmark("round start");
    // SplitMix64 draw counters: accelerated uses b proposal + b accept draws per round
    // (rpcholesky.hpp:362-364, 179), block b proposals (293-296), simple one (226)
    const uint64_t draw0 = (algo == kAlgoAccelerated ? 2ull : 1ull) * (uint64_t)b * (uint64_t)round;
    // -- K2: scan of the residual diagonal (+ previous round's ||G||^2 partials)
    // one shard: the totals pass also runs the chunk prefix (its last CTA), no extra launch
    FusedPrefix fp;
    const bool fuse_prefix = P == 1 && L.ncg <= kFusedPrefixMax;
    if (fuse_prefix) {
      fp.counter = prefix_counter.as<unsigned>();
      fp.n_chunks = L.ncg;
      fp.chunk_end = chunk_end.as<double>();
      fp.status = d_scan;
      fp.g2_all = pending_g2 ? g2_all.as<double>() : nullptr;
    }
    // (skipped when the previous update already chained its scan: chunk ends, thread bases
    // and the round status are current)
    // one shard: the sampler chains the chunk offsets from the chained totals itself
    const bool sampler_prefix = scan_fresh && P == 1 && ctx->world == 1;
    if (scan_fresh) {
      for (size_t si = 0; si < res->shards.size(); ++si) {
        Shard& s = res->shards[si];
        launch_chunk_chain(scan_tsum[si].as<double>(), s.tile_g2.as<double>(), s.n_loc,
                           s.nchunks, tb_all.as<double>() + (size_t)s.chunk0 * kScanThreads,
                           totals_all.as<double>() + s.chunk0, g2_all.as<double>() + s.chunk0,
                           st);
        ++launches;
      }
    }
    for (Shard& s : res->shards) {
      if (scan_fresh) break;
      // (+ the previous update's per-tile ||G||^2 partials -> per-chunk, fixed order)
      launch_chunk_totals(s.u.as<double>(), s.n_loc, s.nchunks, totals_all.as<double>() + s.chunk0, st,
                          pending_g2 && s.n_loc ? s.tile_g2.as<double>() : nullptr,
                          (int)((s.n_loc + 63) / 64), g2_all.as<double>() + s.chunk0, fp,
                          tb_all.as<double>() + (size_t)s.chunk0 * kScanThreads);
      ++launches;
    }
    if (scan_fresh ? !sampler_prefix : !fuse_prefix) {
      allgather(ctx, totals_all.as<double>(), L.cpr);
      if (pending_g2) allgather(ctx, g2_all.as<double>(), L.cpr);
      launch_chunk_prefix(totals_all.as<double>(), pending_g2 ? g2_all.as<double>() : nullptr,
                          L.ncg, chunk_end.as<double>(), d_scan, st);
      ++launches;
    }
    dbg(st, "scan");
    cmark("chunk totals");
    if (replay) {
      const double* ug = res->shards[0].u.as<double>();
      if (P > 1) {
        for (Shard& s : res->shards)
          if (s.n_loc)
            CK(cudaMemcpyAsync(u_all.as<double>() + (size_t)s.gidx * L.cpr * kChunk, s.u.p,
                               sizeof(double) * s.n_loc, cudaMemcpyDeviceToDevice, st));
        allgather(ctx, u_all.as<double>(), (size_t)L.cpr * kChunk);
        ug = u_all.as<double>();
      }
      launch_replay_scan(ug, n, cumsum.as<double>(), d_scan, st);
      ++launches;
    }
    if (ctx->world > 1) CK(cudaMemsetAsync(prop.p, 0, sizeof(double) * b * lay.rec, st));
    // -- K1/K2: b proposals; owners write their records
    for (Shard& s : res->shards) {
      SampleParams sp{};
      sp.u = s.u.as<double>();
      sp.X = s.X.as<double>();
      sp.sqn = s.sqn.as<double>();
      sp.F = lowmem ? nullptr : s.F.as<double>();
      sp.n_loc = s.n_loc;
      sp.n_global = n;
      sp.dpad = dpad;
      sp.ldf = ldf;
      sp.kcur = lowmem ? 0 : (int)kcur;  // lowmem: factor rows are formed after selection
      sp.row0 = s.row0;
      sp.chunk0 = s.chunk0;
      sp.n_chunks_local = s.nchunks;
      sp.n_chunks_global = L.ncg;
      sp.shard = s.gidx;
      sp.n_shards = P;
      sp.shard_chunk0 = shard_c0.as<int>();
      sp.chunk_end = chunk_end.as<double>();
      sp.seed = cfg.seed;
      sp.draw0 = draw0;
      sp.b = b;
      sp.lay = lay;
      sp.records = prop.as<double>();  // the owner of draw j writes slot j
      sp.owner = owner.as<int>();
      sp.tb = tb_all.as<double>() + (size_t)s.chunk0 * kScanThreads;
      if (sampler_prefix) {  // (one shard) offsets + status from the update's chunk totals
        sp.totals = totals_all.as<double>();
        sp.chunk_g2 = g2_all.as<double>();
        sp.chunk_end_out = chunk_end.as<double>();
        sp.status = d_scan;
      }
      // every shard runs the sampler, including shards without rows (it returns early for
      // draws it does not own)
      if (replay) launch_replay_sample(sp, cumsum.as<double>(), st);
      else launch_sample(sp, st);
      dbg(st, "sample");
      ++launches;
    }
    cmark("sample");
    allreduce_owner(ctx, prop.p, (size_t)b * lay.rec);
    if (lowmem && kcur > 0) {
      // F(S', :) = A(S', S) L^{-T}  (= W_prop^T of rpcholesky.hpp:441-444)
      launch_kprop(prop.as<double>(), lay, b, piv.as<double>(), prec, (int)kcur, (int)d, kind, kfun,
                   kspec.sigma, Kp.as<double>(), ldf, st);
      launch_gemm(b, (int)kcur, (int)kcur, 1.0, Kp.as<double>(), ldf, 0, Linv.as<double>(), ldf, 1,
                  0.0, prop.as<double>() + lay.foff, lay.rec, st);
      launches += 2;
      dbg(st, "lowmem fprop");
    }
    auto h_wake = clk::now();  // (RPC_DEBUG_CHAIN) the host learned the round's status
    if (algo != kAlgoAccelerated) {
      // ---- block_rpcholesky (rpcholesky.hpp:268-333) / simple_rpcholesky (206-246):
      // every distinct proposal is kept (sorted), its block factored by an all-accepting
      // sweep (= LLT: fails on a pivot <= 0); block retries once with a diagonal shift.
      CK(cudaMemcpyAsync(hbuf, status.p, sizeof(ScanStatus), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpy2DAsync(h_prop_ids, sizeof(double), prop.p, lay.rec * sizeof(double),
                           sizeof(double), b, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaGetLastError());
      if (pending_g2) {
        captured_sq += h_scan->g2_prev;
        pending_g2 = false;
      }
      if (h_scan->exhausted) {
        res->exhausted = true;
        break;
      }
      if (algo == kAlgoBlock && cfg.stop_tol > 0.0 &&
          (trace_a - captured_sq) <= cfg.stop_tol * trace_a)
        break;
      // kept = unique_sorted(proposed) (rpcholesky.hpp:297); record of its first draw
      std::vector<std::pair<int64_t, int>> ids(b);
      for (int j = 0; j < b; ++j) ids[j] = {(int64_t)h_prop_ids[j], j};
      std::sort(ids.begin(), ids.end());
      std::vector<int> kidx;
      for (int j = 0; j < b; ++j)
        if (j == 0 || ids[j].first != ids[j - 1].first) kidx.push_back(ids[j].second);
      const int mk = (int)kidx.size();
      CK(cudaMemcpyAsync(kept_idx.p, kidx.data(), sizeof(int) * mk, cudaMemcpyHostToDevice, st));
      launch_gather_records(prop.as<double>(), lay.rec, 2 + dpad + kcur, kept_idx.as<int>(), mk,
                            propk.as<double>(), st);
      launch_hblock(propk.as<double>(), lay, mk, (int)dpad, (int)d, (int)kcur, kind, kfun, kspec.sigma,
                    Hbuf.as<double>(), st, hb_part.as<double>(), hb_tick.as<unsigned>());
      launches += 2;
      for (int attempt = 0;; ++attempt) {
        launch_sweep(Hbuf.as<double>(), mk, cfg.seed, 0, propk.as<double>(), lay, pos.as<int>(),
                     acc_ids.as<int64_t>(), lcol.as<double>(), lacc.as<double>(), d_sweep,
                     hp.as<double>(), st, 1);
        ++launches;
        CK(cudaMemcpyAsync(h_sweep, d_sweep, sizeof(SweepOut), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h_sweep->m == mk) break;
        if (algo == kAlgoSimple) break;  // !(g[s] > 0): rank exhausted (rpcholesky.hpp:229-232)
        if (attempt == 1)
          raise(RPC_ENUMERIC, "block_rpcholesky: Cholesky failed after diagonal shift");
        // shift = 64 eps tr(A) / N (rpcholesky.hpp:313-315); tr(A) = N for kernel oracles
        launch_add_diag(Hbuf.as<double>(), mk, 64.0 * 2.220446049250313e-16 * trace_a / (double)n, st);
        ++launches;
      }
      if (algo == kAlgoSimple && h_sweep->m != mk) {
        res->exhausted = true;
        break;
      }
      if (!grouped) {
        CK(cudaMemsetAsync(linv.p, 0, sizeof(double) * nbl * ldl, st));
        launch_linv(lacc.as<double>(), mk, (int)nbl, ldl, (int)(kcur & 1), linv.as<double>(), st);
        launch_gather_accepted(propk.as<double>(), lay, pos.as<int>(), mk, 256, 0, (int)dpad,
                               xs.as<double>(), fs.as<double>(), ldf, sqnS.as<double>(),
                               idS.as<double>(), st, nullptr, gram_xscale(kind));
        launch_bprime(linv.as<double>(), ldl, (int)(kcur & 1), propk.as<double>(), lay,
                      pos.as<int>(), &d_sweep->m, mk, (int)kcur, fs.as<double>(), ldf, st);
        launches += 3;
      }
      CK(cudaMemcpyAsync(h_acc_ids, acc_ids.p, sizeof(int64_t) * mk, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else {
    // -- K3: H block; K4: rejection sweep (replicated on every shard)
    launch_hblock(prop.as<double>(), lay, b, (int)dpad, (int)d, (int)kcur, kind, kfun, kspec.sigma,
                  Hbuf.as<double>(), st, hb_part.as<double>(), hb_tick.as<unsigned>());
    dbg(st, "hblock");
    cmark("hblock");
    // the sweep's tail also publishes the round status into mapped host memory
    // (fused: the round prep runs in the same launch behind the sweep, and the host spins on
    // the status's sequence word instead of an event)
    bool fused = false;
    const unsigned epoch = next_epoch();
    if (fused_prep_ok && hbuf_dev && !grouped && !lowmem && b <= 128) {
      const int g = launch_sweep_prep(
          Hbuf.as<double>(), b, cfg.seed, draw0 + (uint64_t)b, prop.as<double>(), lay,
          pos.as<int>(), acc_ids.as<int64_t>(), lcol.as<double>(), lacc.as<double>(), d_sweep,
          d_scan, hbuf_dev, sweep_prog.as<unsigned long long>(), sweep_aidx.as<int>(), epoch,
          (int)nbl, ldl, linv.as<double>(), (int)kcur, fs.as<double>(), ldf, (int)dpad,
          xs.as<double>(), sqnS.as<double>(), idS.as<double>(), gram_xscale(kind), 256, st);
      if (g < 0 && g != -3) CK(cudaGetLastError());
      fused = g > 0;
    }
    if (!fused)
      launch_sweep(Hbuf.as<double>(), b, cfg.seed, draw0 + (uint64_t)b, prop.as<double>(), lay,
                   pos.as<int>(), acc_ids.as<int64_t>(), lcol.as<double>(), lacc.as<double>(),
                   d_sweep, hp.as<double>(), st, 0, hbuf_dev ? d_scan : nullptr, hbuf_dev);
    dbg(st, "sweep");
    cmark("sweep");
    launches += 2;
    if (hbuf_dev) {
      // status words went straight into mapped host memory (sweep tail): no copy-engine
      // transfer, so the read never queues behind a factor block streaming out on the copy
      // stream; recorded before L^{-1} / B' so the host's bookkeeping overlaps them and the
      // update kernel is already queued when they finish.
      CK(cudaEventRecord(ev_pub.e, st));
    }
    // L^{-1} and the accepted-pivot operands only need the sweep's device-side outputs:
    // queue them before the status read so they run while the host waits (grouped rounds
    // build them per group once m is known).
    if (!grouped && !fused) {
      // (no memset of the L^{-1} buffer: both kernels write every row of every column the
      // consumers read, zeros included)
      if (lowmem) {
        launch_linv_dev(lacc.as<double>(), &d_sweep->m, b, (int)nbl, ldl, 0, linv.as<double>(), st, 0);
        ++launches;
      } else {
        // L^{-1}, B' (by substitution, beside L^{-1}) and the accepted operands: one launch
        // (was linv -> gather -> bprime: C4 43.03 -> 42.77 ms, C1 0.71 -> 0.63 ms)
        launch_round_prep(lacc.as<double>(), 0, &d_sweep->m, b, (int)nbl, ldl, (int)(kcur & 1),
                          linv.as<double>(), prop.as<double>(), lay, pos.as<int>(), (int)kcur,
                          fs.as<double>(), ldf, (int)dpad, xs.as<double>(), sqnS.as<double>(),
                          idS.as<double>(), gram_xscale(kind), 256, st);
        ++launches;
      }
    }
    cmark("round prep");
    if (dbg_gaps) {  // RPC_DEBUG_GAPS: device idle between the round prep and the update
      gap_ev.emplace_back();
      CK(cudaEventRecord(gap_ev.back().e, st));
    }
    if (hbuf_dev) {
      // (published right after the sweep, above)
    } else {
      CK(cudaMemcpyAsync(hbuf, status.p, sizeof(ScanStatus) + sizeof(SweepOut),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpy2DAsync(h_prop_ids, sizeof(double), prop.p, lay.rec * sizeof(double),
                           sizeof(double), b, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_acc_ids, acc_ids.p, sizeof(int64_t) * b, cudaMemcpyDeviceToHost, st));
    }
    if (fused) wait_published(&h_sweep->pad, epoch, ev_pub.e);
    else if (hbuf_dev) CK(cudaEventSynchronize(ev_pub.e));
    else CK(cudaStreamSynchronize(st));
    h_wake = clk::now();
    }  // accelerated
    CK(cudaGetLastError());
    if (pending_g2) {
      captured_sq += h_scan->g2_prev;  // captured_sq += ||G||_F^2 (rpcholesky.hpp:388)
      pending_g2 = false;
    }
    if (h_scan->exhausted) {  // rpcholesky.hpp:356-359
      res->exhausted = true;
      break;
    }
    if (cfg.stop_tol > 0.0 && (trace_a - captured_sq) <= cfg.stop_tol * trace_a) break;
    const int m = h_sweep->m;
    std::vector<int64_t> pr(b), ac(m);
    for (int j = 0; j < b; ++j) pr[j] = (int64_t)h_prop_ids[j];
    for (int a = 0; a < m; ++a) ac[a] = h_acc_ids[a];
    if (m > 0) {
      if (kcur + m > cap)
        raise(RPC_ENUMERIC, "accelerated_rpcholesky: factor capacity exceeded (duplicate pivot)");
      // (block / simple: kept blocks have m <= b, so cap = min(N, k + b) always suffices)
      // (g2_all needs no per-round reset: every round writes the same chunk slots, and the
      // slots no shard writes stay zero from setup)
      if (lowmem) {
        // L_new = [[L, 0], [F_S, L_sel]]; L_new^{-1} rows [kcur, kcur+m) =
        // [-L_sel^{-1} (F_S L^{-1}) | L_sel^{-1}]   (rpcholesky.hpp:470-475)
        launch_lowmem_append(prop.as<double>(), lay, pos.as<int>(), m, (int)kcur, prec,
                             lacc.as<double>(), linv.as<double>(), ldl, piv.as<double>(),
                             fsl.as<double>(), ldf, Lrm.as<double>(), Linv.as<double>(), ldf, st);
        ++launches;
        if (kcur > 0) {
          launch_gemm(m, (int)kcur, (int)kcur, 1.0, fsl.as<double>(), ldf, 0, Linv.as<double>(),
                      ldf, 0, 0.0, T1.as<double>(), ldf, st);
          launch_gemm(m, (int)kcur, m, -1.0, Linv.as<double>() + kcur * ldf + kcur, ldf, 0,
                      T1.as<double>(), ldf, 0, 0.0, Linv.as<double>() + kcur * ldf, ldf, st);
          launches += 2;
        }
        dbg(st, "lowmem append");
        for (Shard& s : res->shards) {
          if (s.n_loc == 0) continue;
          LowmemParams lp{};
          lp.X = s.X.as<double>();
          lp.dpad = dpad;
          lp.dchunks = (int)(dpad / 16);
          lp.d = (int)d;
          lp.sqn = s.sqn.as<double>();
          lp.u = s.u.as<double>();
          lp.n_loc = s.n_loc;
          lp.row0 = s.row0;
          lp.piv = piv.as<double>();
          lp.prec = prec;
          lp.W = Linv.as<double>() + kcur * ldf;
          lp.ldw = ldf;
          lp.m = m;
          lp.kold = (int)kcur;
          lp.knew = (int)(kcur + m);
          lp.kind = kind;
          lp.kfun = kernel_fun(kspec, &lp.escale);
          lp.tile_g2 = s.tile_g2.as<double>();
          lp.pin = 1;
          upd_ev.emplace_back();
          upd_ev.emplace_back();
          CK(cudaEventRecord(upd_ev[upd_ev.size() - 2].e, st));
          const int bm = launch_lowmem(lp, st);
          CK(cudaEventRecord(upd_ev.back().e, st));
          dbg(st, "lowmem update");
          if (bm < 0)
            raise(RPC_ECUDA, "low-memory update launch failed (code " + std::to_string(bm) + ")");
          launches += 1;  // per-tile ||G||^2 -> chunks: folded into the next chunk-totals pass
          ++upd_launches;
          const double N = (double)s.n_loc, kn = (double)(kcur + m);
          const double fl = 2.0 * N * m * kn + (kind == kGaussGram ? 2.0 * N * kn * d : 0.0);
          flops += fl;
          upd_info.emplace_back(m, kcur);
          upd_flops.push_back(fl);
          bytes += 8.0 * (N * d + 2.0 * N);
        }
      }
      const double* recs = algo == kAlgoAccelerated ? prop.as<double>() : propk.as<double>();
      // balanced groups of at most kGroup pivots (multiples of 8 but the last)
      const int ngroups = grouped ? (m + kGroup - 1) / kGroup : 1;
      const int gsz = grouped ? (int)round_up((m + ngroups - 1) / ngroups, 8) : m;
      for (int g0 = 0; g0 < m && !lowmem; g0 += gsz) {
      const int mg = std::min(gsz, m - g0);
      const int64_t kg = kcur + g0;  // F columns already holding earlier groups of this round
      if (grouped) {
        CK(cudaMemcpy2DAsync(lsub.p, sizeof(double) * mg, lacc.as<double>() + (int64_t)g0 * m + g0,
                             sizeof(double) * m, sizeof(double) * mg, mg, cudaMemcpyDeviceToDevice,
                             st));
        CK(cudaMemsetAsync(linv.p, 0, sizeof(double) * nbl * ldl, st));
        launch_linv(lsub.as<double>(), mg, (int)nbl, ldl, (int)(kg & 1), linv.as<double>(), st);
        launch_gather_accepted(recs, lay, pos.as<int>() + g0, mg, 256, (int)kg, (int)dpad,
                               xs.as<double>(), fs.as<double>(), ldf, sqnS.as<double>(),
                               idS.as<double>(), st, nullptr, gram_xscale(kind));
        launch_bprime(linv.as<double>(), ldl, (int)(kg & 1), recs, lay, pos.as<int>() + g0, nullptr,
                      mg, (int)kg, fs.as<double>(), ldf, st, lacc.as<double>(), m, g0, (int)kcur);
        launches += 3;
      }
      for (Shard& s : res->shards) {
        if (s.n_loc == 0 || lowmem) continue;
        UpdateParams up{};
        up.X = s.X.as<double>();
        up.dpad = dpad;
        up.dchunks = (int)(dpad / 16);
        up.d = (int)d;
        up.sqn = s.sqn.as<double>();
        up.F = s.F.as<double>();
        up.ldf = ldf;
        up.kcur = (int)kg;
        up.u = s.u.as<double>();
        up.n_loc = s.n_loc;
        up.row0 = s.row0;
        up.xs = xs.as<double>();
        up.fs = fs.as<double>();
        up.ldfs = ldf;
        up.sqnS = sqnS.as<double>();
        up.idS = idS.as<double>();
        up.m = mg;
        up.linv = linv.as<double>();
        up.ldl = ldl;
        up.sigma = kspec.sigma;
        up.kind = kind;
        up.kfun = kernel_fun(kspec, &up.escale);
        up.tile_g2 = s.tile_g2.as<double>();
        up.g2_accum = g0 > 0;  // later groups add their ||G||^2 to the round's tile partials
        const bool fscan = fuse_scan_ok && !grouped && algo == kAlgoAccelerated &&
                           update_regp2(mg) && update_tile_rows(mg) == 64;
        if (fscan) up.tsum = scan_tsum[&s - res->shards.data()].as<double>();

        scan_fresh = fscan;
        if (dbg_trace) {
          CK(cudaMemsetAsync(trace_buf.p, 0, trace_buf.bytes, st));
          up.trace = trace_buf.as<unsigned long long>();
        }
        if (dbg_phase) {
          CK(cudaMemsetAsync(phase_clk.p, 0, phase_clk.bytes, st));
          up.phase_clk = phase_clk.as<unsigned long long>();
        }
        const bool use_i8 = i8_ok && kg >= i8_min_k && mg <= kI8MaxCols && mg >= kI8MinCols;
        if (use_i8 && slice_pending) {  // the planes must hold every column below kg
          CK(cudaStreamWaitEvent(st, ev_slice_done.e, 0));  // (ahead of the update's timing events)
          slice_pending = false;
        }
        upd_ev.emplace_back();
        upd_ev.emplace_back();
        CK(cudaEventRecord(upd_ev[upd_ev.size() - 2].e, st));
        // (the tensor-core residual GEMM is timed as part of the round's update)
        // (the int8 product costs as much as 64 columns whatever m is: small groups stay on DMMA)
        if (use_i8) {
          const size_t si = &s - res->shards.data();
          tc_ev.emplace_back();
          tc_ev.emplace_back();
          CK(cudaEventRecord(tc_ev[tc_ev.size() - 2].e, st));
          if (launch_i8_residual(reinterpret_cast<const int8_t*>(i8_planes[si].p), i8_rows[si],
                                 i8_kcap, s.n_loc, fs.as<double>(), ldf, mg, (int)kg,
                                 reinterpret_cast<int8_t*>(i8_bplanes.p), i8_cscale.as<double>(),
                                 i8_c.as<double>(), kI8MaxCols, st) == 0) {
            up.cext = i8_c.as<double>();
            up.ldce = kI8MaxCols;
            ++i8_launches;
            launches += 2;
            // products as issued: N = 64 per column half (m <= 64), else m rounded up to 16
            const double rows = (double)round_up(s.n_loc, 128),
                         cols = (double)(mg <= 64 ? 64 : round_up(mg, 16));
            tc_ops += 2.0 * (kI8Slices * (kI8Slices + 1) / 2) * rows * cols * (double)round_up(kg, 64);
            tc_fl += 2.0 * (double)s.n_loc * mg * (double)kg;
          }
          CK(cudaEventRecord(tc_ev.back().e, st));
        }
        if (dbg_chain) host_pre_us += 1e3 * ms_since(h_wake);
        cmark("host gap");
        const auto h_l0 = clk::now();
        const int bm = launch_update(up, st);
        if (dbg_chain) host_launch_us += 1e3 * ms_since(h_l0);
        CK(cudaEventRecord(upd_ev.back().e, st));
        dbg(st, "update");
        cmark("update");
        if (dbg_phase) {
          std::vector<unsigned long long> h(phase_clk.bytes / 8);
          CK(cudaMemcpyAsync(h.data(), phase_clk.p, phase_clk.bytes, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          double sum[8] = {0};
          int nb = 0;
          for (size_t b = 0; b < h.size() / 8; ++b) {
            if (!h[b * 8 + 5]) continue;
            ++nb;
            for (int q = 0; q < 8; ++q) sum[q] += (double)h[b * 8 + q];
          }
          std::fprintf(stderr,
                       "[rpc] phases m=%d kcur=%lld (Mcycles/CTA): X %.3f drain %.3f sqn %.3f exp %.3f F %.3f "
                       "park %.3f trsm %.3f epi %.3f\n",
                       m, (long long)kcur, sum[0] / nb / 1e6, sum[6] / nb / 1e6, sum[7] / nb / 1e6,
                       sum[1] / nb / 1e6,
                       sum[2] / nb / 1e6, sum[3] / nb / 1e6, sum[4] / nb / 1e6, sum[5] / nb / 1e6);
        }
        if (dbg_trace) dump_trace(trace_buf, m, kcur, st);
        if (bm < 0) raise(RPC_ECUDA, "update kernel launch failed (code " + std::to_string(bm) + ")");
        launches += 1;  // per-tile ||G||^2 -> chunks: folded into the next chunk-totals pass
        ++upd_launches;
        const double N = (double)s.n_loc;
        const double fl = 2.0 * N * mg * kg + N * (double)mg * mg + 2.0 * N * mg * d;
        flops += fl;
        upd_info.emplace_back(mg, kg);
        upd_flops.push_back(fl);
        bytes += 8.0 * (N * kg + N * mg + N * d + 2.0 * N);
      }
      // this group's columns into F's digit planes (coalesced: a warp per row segment; byte
      // stores from the update epilogue's fragment layout measured 3-4x slower per round): the
      // next group's (or round's) residual GEMM reads them
      // (not after the last group of the last round: nothing reads its digits)
      const bool last_round = cfg.mode == RPC_FIXED_ROUNDS ? round + 1 >= cfg.rounds
                                                           : kcur + m >= cfg.target_rank;
      if (i8_ok && !(last_round && g0 + mg >= m)) {
        sl_ev.emplace_back();
        sl_ev.emplace_back();
        if (ast != st) {
          CK(cudaEventRecord(ev_upd_done.e, st));
          CK(cudaStreamWaitEvent(ast, ev_upd_done.e, 0));
        }
        CK(cudaEventRecord(sl_ev[sl_ev.size() - 2].e, ast));
        for (size_t si = 0; si < res->shards.size(); ++si) {
          Shard& s = res->shards[si];
          launch_slice_cols(s.F.as<double>(), ldf, s.n_loc, (int)kg, mg,
                            reinterpret_cast<int8_t*>(i8_planes[si].p), i8_rows[si], i8_kcap, ast);
          ++launches;
        }
        CK(cudaEventRecord(sl_ev.back().e, ast));
        if (ast != st) {
          CK(cudaEventRecord(ev_slice_done.e, ast));
          slice_pending = true;
        }
      }
      }  // groups
      pending_g2 = true;
      if (sink.p) {
        const auto hs0 = clk::now();
        CK(cudaEventRecord(sink_ev[sink_slot].e, st));
        CK(cudaStreamWaitEvent(cst, sink_ev[sink_slot].e, 0));
        int64_t off = 0;
        for (Shard& s : res->shards) {
          if (s.n_loc == 0) continue;
          double* tmp = sink_tmp[sink_slot].as<double>() + off;
          launch_f_to_colmajor(s.F.as<double>(), ldf, s.n_loc, (int)kcur, m, tmp, s.n_loc, cst);
          CK(cudaMemcpy2DAsync(sink.p + kcur * sink.ld + s.row0, sink.ld * sizeof(double), tmp,
                               s.n_loc * sizeof(double), s.n_loc * sizeof(double), m,
                               cudaMemcpyDeviceToHost, cst));
          off += s.n_loc * m;
          ++launches;
        }
        if (std::getenv("RPC_DEBUG_TIMING"))
          std::fprintf(stderr, "[rpc] sink round %lld: host enqueue %.3f ms\n", (long long)round,
                       ms_since(hs0));
        sink_slot ^= 1;
      }
      res->pivots.insert(res->pivots.end(), ac.begin(), ac.end());
      kcur += m;
    }
    res->proposed.push_back(std::move(pr));
    res->accepted.push_back(std::move(ac));
  }
  if (slice_pending) CK(cudaStreamWaitEvent(st, ev_slice_done.e, 0));
  CK(cudaEventRecord(ev_t1.e, st));
  if (sink.p) CK(cudaStreamSynchronize(cst));  // every column is on the host
  const double loop_ms = ms_since(h1);
  const auto h2 = clk::now();
  // ---- finalize ----------------------------------------------------------------
  NvtxRange nv_fin("rpc:finalize");
  if (pending_g2) {  // last round's ||G||^2 (no further scan consumed it)
    for (Shard& s : res->shards) {
      if (s.n_loc == 0) continue;
      launch_tile_to_chunk(s.tile_g2.as<double>(), (int)((s.n_loc + 63) / 64), kChunk / 64,
                           s.nchunks, g2_all.as<double>() + s.chunk0, st);
      ++launches;
    }
    allgather(ctx, g2_all.as<double>(), L.cpr);
    launch_chunk_prefix(totals_all.as<double>(), g2_all.as<double>(), L.ncg,
                        chunk_end.as<double>(), d_scan, st);
    ++launches;
    CK(cudaMemcpyAsync(hbuf, status.p, sizeof(ScanStatus), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    captured_sq += h_scan->g2_prev;
  }
  res->kcur = kcur;
  res->captured_sq = captured_sq;
  if (cfg.mode == RPC_UNTIL_RANK && kcur > cfg.target_rank) res->surplus = kcur - cfg.target_rank;
  // ||F||_F^2 for relative_trace_error (rpcholesky.hpp:577-583): the factor's squared
  // Frobenius norm is the sum over rounds of ||G_r||_F^2, already reduced in a fixed
  // chunk order per round, so no extra pass over the N x k factor is needed.
  res->fro2 = captured_sq;
  // chol_factor = lower(F(pivots, :)) (rpcholesky.hpp:140-145): owners gather pivot rows
  // into a device-resident column-major k x k buffer; copied out on request.
  if (kcur > 0 && lowmem) {
    res->chol_dev = DBuf(ctx, sizeof(double) * kcur * kcur);
    launch_lowmem_chol(Lrm.as<double>(), ldf, (int)kcur, res->chol_dev.as<double>(), st);
    ++launches;
    CK(cudaStreamSynchronize(st));
  } else if (kcur > 0) {
    DBuf piv(ctx, sizeof(int64_t) * kcur);
    res->chol_dev = DBuf(ctx, sizeof(double) * kcur * kcur);
    CK(cudaMemcpyAsync(piv.p, res->pivots.data(), sizeof(int64_t) * kcur, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(res->chol_dev.p, 0, sizeof(double) * kcur * kcur, st));
    for (Shard& s : res->shards) {
      if (s.n_loc == 0) continue;
      chol_gather_kernel<<<(unsigned)kcur, 128, 0, st>>>(s.F.as<double>(), ldf, s.row0, s.n_loc,
                                                          piv.as<int64_t>(), kcur,
                                                          res->chol_dev.as<double>());
      ++launches;
    }
    // each pivot row lives on exactly one rank: the owner reduce keeps its words
    allreduce_owner(ctx, res->chol_dev.p, (size_t)kcur * kcur);
    CK(cudaStreamSynchronize(st));  // piv returns to the pool
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev_t0.e, ev_t1.e));
  tm.factorize_ms = ms;
  CK(cudaEventElapsedTime(&ms, ev_up0.e, ev_up1.e));
  tm.upload_ms = ms;
  const bool dbg_timing = std::getenv("RPC_DEBUG_TIMING") != nullptr;
  for (size_t i = 0; i + 1 < upd_ev.size(); i += 2) {
    CK(cudaEventElapsedTime(&ms, upd_ev[i].e, upd_ev[i + 1].e));
    update_ms += ms;
    if (dbg_timing && i / 2 < upd_info.size())
      std::fprintf(stderr, "[rpc] update %zu: m=%d kcur=%lld  %.3f ms  %.2f TF/s\n", i / 2,
                   upd_info[i / 2].first, (long long)upd_info[i / 2].second, ms,
                   upd_flops[i / 2] / (ms * 1e-3) / 1e12);
  }
  tm.update_ms = update_ms;
  if (dbg_gaps && !upd_ev.empty()) {
    // pairs (prep done, update start): the host's per-round work showing up as device idle
    double tot = 0.0;
    for (size_t i = 0; i < gap_ev.size() && 2 * i < upd_ev.size(); ++i) {
      CK(cudaEventElapsedTime(&ms, gap_ev[i].e, upd_ev[2 * i].e));
      tot += ms;
      std::fprintf(stderr, "[rpc] round %zu: prep end -> update start %.3f ms\n", i, ms);
    }
    std::fprintf(stderr, "[rpc] total prep->update gap %.3f ms\n", tot);
  }
  if (dbg_chain && chain_ev.size() > 1) {
    std::vector<std::pair<std::string, std::pair<double, int>>> agg;
    for (size_t i = 1; i < chain_ev.size(); ++i) {
      CK(cudaEventElapsedTime(&ms, chain_ev[i - 1].second.e, chain_ev[i].second.e));
      std::string lab = chain_ev[i].first;
      auto it = std::find_if(agg.begin(), agg.end(), [&](auto& a) { return a.first == lab; });
      if (it == agg.end()) agg.push_back({lab, {ms, 1}});
      else it->second.first += ms, it->second.second += 1;
    }
    for (auto& a : agg)
      std::fprintf(stderr, "[rpc] chain %-14s %4d x  avg %8.1f us  total %8.3f ms\n",
                   a.first.c_str(), a.second.second, 1e3 * a.second.first / a.second.second,
                   a.second.first);
    std::fprintf(stderr, "[rpc] host: wake -> update launch %.1f us, launch call %.1f us (per update)\n",
                 host_pre_us / std::max<int64_t>(1, upd_launches),
                 host_launch_us / std::max<int64_t>(1, upd_launches));
  }
  {
    double tcm = 0.0, slm = 0.0;
    for (size_t i = 0; i + 1 < tc_ev.size(); i += 2) {
      CK(cudaEventElapsedTime(&ms, tc_ev[i].e, tc_ev[i + 1].e));
      tcm += ms;
    }
    for (size_t i = 0; i + 1 < sl_ev.size(); i += 2) {
      CK(cudaEventElapsedTime(&ms, sl_ev[i].e, sl_ev[i + 1].e));
      slm += ms;
    }
    tm.tc_ms = tcm;
    tm.tc_int8_ops = tc_ops;
    tm.tc_fp64_flops = tc_fl;
    tm.tc_slice_ms = slm;
  }
  tm.update_flops = flops;
  tm.update_bytes = bytes;
  tm.update_launches = upd_launches;
  tm.kernel_launches = launches;
  tm.host_setup_ms = setup_ms;
  tm.host_loop_ms = loop_ms;
  tm.host_final_ms = ms_since(h2);
  tm.host_total_ms = ms_since(h0);
  // release the point copies; F, u stay with the result
  for (Shard& s : res->shards) {
    s.X.release();
    s.sqn.release();
    s.tile_g2.release();
  }
}

rpc_result* new_result() { return new rpc_result(); }

}  // namespace rpcb_rt

using namespace rpcb_rt;

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* rpc_last_error(const rpc_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

static int make_ctx(int device, int nvirt, rpc_ctx** out) {
  if (!out) return fail(nullptr, RPC_EINVAL, "null output pointer");
  *out = nullptr;
  rpc_ctx* ctx = new rpc_ctx();
  int rc = guarded(ctx, [&] {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) raise(RPC_ECUDA, "rpc_create: no such CUDA device");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) raise(RPC_ECUDA, "rpc_create: this build targets sm_100a (B200)");
    if (nvirt < 1 || nvirt > 64) raise(RPC_EINVAL, "rpc_create_virtual: n_shards must be in [1, 64]");
    ctx->device = device;
    ctx->nvirt = nvirt;
    CK(cudaSetDevice(device));
    // the main stream outranks the copy and append streams: the round chain's small kernels
    // are scheduled ahead of the blocks those streams still have queued
    int prio_least = 0, prio_greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    CK(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, prio_greatest));
    CK(cudaStreamCreateWithPriority(&ctx->copy_stream, cudaStreamNonBlocking, prio_least));
    CK(cudaStreamCreateWithPriority(&ctx->aux_stream, cudaStreamNonBlocking, prio_least));
  });
  if (rc) {
    g_last_error = ctx->err;
    delete ctx;
    return rc;
  }
  *out = ctx;
  return RPC_OK;
}

int rpc_create(int device, rpc_ctx** out) { return make_ctx(device, 1, out); }
int rpc_create_virtual(int device, int n_shards, rpc_ctx** out) {
  return make_ctx(device, n_shards, out);
}

int rpc_nccl_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
  });
}

int rpc_create_nccl(int device, const void* id128, int nranks, int rank, rpc_ctx** out) {
  int rc = make_ctx(device, 1, out);
  if (rc) return rc;
  rpc_ctx* ctx = *out;
  rc = guarded(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) raise(RPC_EINVAL, "rpc_create_nccl: bad rank");
    ctx->world = nranks;
    ctx->rank = rank;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(&id, id128, sizeof id);
      NK(ncclCommInitRank(&ctx->comm, nranks, id, rank));
    }
  });
  if (rc) {
    g_last_error = ctx->err;
    rpc_destroy(ctx);
    *out = nullptr;
  }
  return rc;
}

int rpc_create_hostcoll(int device, int nranks, int rank, const rpc_host_collectives* ops,
                        rpc_ctx** out) {
  if (!ops || !ops->allgather || !ops->allreduce_or_u64)
    return fail(nullptr, RPC_EINVAL, "rpc_create_hostcoll: missing collective callbacks");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(nullptr, RPC_EINVAL, "rpc_create_hostcoll: bad rank");
  int rc = make_ctx(device, 1, out);
  if (rc) return rc;
  rpc_ctx* ctx = *out;
  ctx->world = nranks;
  ctx->rank = rank;
  ctx->hostcoll = true;
  ctx->hc = *ops;
  return RPC_OK;
}

void rpc_destroy(rpc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto fn : ctx->on_destroy) fn(ctx);
  ctx->trim();
  if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
  if (ctx->io_pinned) cudaFreeHost(ctx->io_pinned);
  if (ctx->hc_pinned) cudaFreeHost(ctx->hc_pinned);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
  delete ctx;
}

int rpc_plan_shards(int64_t n, int n_shards, int shard, int64_t* row0, int64_t* nrows,
                    int* chunk0, int* nchunks, int* chunks_per_shard) {
  if (n < 1 || n_shards < 1 || shard < 0 || shard >= n_shards)
    return fail(nullptr, RPC_EINVAL, "rpc_plan_shards: bad arguments");
  const Layout L = make_layout(n, n_shards);
  if (row0) *row0 = L.row0(shard);
  if (nrows) *nrows = L.rows(shard);
  if (chunk0) *chunk0 = shard * L.cpr;
  if (nchunks) *nchunks = L.chunks(shard);
  if (chunks_per_shard) *chunks_per_shard = L.cpr;
  return RPC_OK;
}

int rpc_shard_rows(const rpc_ctx* ctx, int64_t n, int local, int64_t* row0, int64_t* nrows) {
  if (!ctx || local < 0 || local >= ctx->nvirt || n < 0) return RPC_EINVAL;
  const Layout L = make_layout(n, ctx->nshards());
  const int s = ctx->first_shard() + local;
  *row0 = L.row0(s);
  *nrows = L.rows(s);
  return RPC_OK;
}

int rpc_accelerated_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                               int layout, rpc_kernel_spec kernel, rpc_run_config cfg,
                               rpc_result** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  int rc = guarded(ctx, [&] {
    if (!x && n > 0) raise(RPC_EINVAL, "null point matrix");
    if (ldx < (layout == RPC_ROW_MAJOR ? d : n)) raise(RPC_EINVAL, "leading dimension too small");
    run_factorization(ctx, x, false, n, d, ldx, layout, kernel, cfg, r);
  });
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

int rpc_accelerated_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                      int64_t ldx, int layout, rpc_kernel_spec kernel,
                                      rpc_run_config cfg, rpc_result** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  int rc = guarded(ctx, [&] { run_factorization(ctx, x_dev, true, n, d, ldx, layout, kernel, cfg, r); });
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

int rpc_accelerated_rpcholesky_lowmem(rpc_ctx* ctx, const double* x, int64_t n, int64_t d,
                                      int64_t ldx, int layout, rpc_kernel_spec kernel,
                                      rpc_run_config cfg, rpc_result** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  int rc = guarded(ctx, [&] {
    if (!x && n > 0) raise(RPC_EINVAL, "null point matrix");
    if (ldx < (layout == RPC_ROW_MAJOR ? d : n)) raise(RPC_EINVAL, "leading dimension too small");
    if (cfg.block_size < 1)
      raise(RPC_EINVAL, "accelerated_rpcholesky_lowmem: block size must be >= 1");
    run_factorization(ctx, x, false, n, d, ldx, layout, kernel, cfg, r, true);
  });
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

int rpc_accelerated_rpcholesky_lowmem_device(rpc_ctx* ctx, const double* x_dev, int64_t n,
                                             int64_t d, int64_t ldx, int layout,
                                             rpc_kernel_spec kernel, rpc_run_config cfg,
                                             rpc_result** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  int rc = guarded(ctx, [&] {
    if (cfg.block_size < 1)
      raise(RPC_EINVAL, "accelerated_rpcholesky_lowmem: block size must be >= 1");
    run_factorization(ctx, x_dev, true, n, d, ldx, layout, kernel, cfg, r, true);
  });
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

static int run_algo(rpc_ctx* ctx, const double* x, bool on_device, int64_t n, int64_t d,
                    int64_t ldx, int layout, rpc_kernel_spec kernel, rpc_run_config cfg, int algo,
                    rpc_result** out) {
  if (!ctx || !out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  int rc = guarded(ctx, [&] {
    if (!x && n > 0) raise(RPC_EINVAL, "null point matrix");
    if (!on_device && ldx < (layout == RPC_ROW_MAJOR ? d : n))
      raise(RPC_EINVAL, "leading dimension too small");
    run_factorization(ctx, x, on_device, n, d, ldx, layout, kernel, cfg, r, false, algo);
  });
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

int rpc_block_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                         int layout, rpc_kernel_spec kernel, rpc_run_config cfg, rpc_result** out) {
  if (cfg.block_size < 1) return fail(ctx, RPC_EINVAL, "block_rpcholesky: block size must be >= 1");
  return run_algo(ctx, x, false, n, d, ldx, layout, kernel, cfg, kAlgoBlock, out);
}

int rpc_block_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                int64_t ldx, int layout, rpc_kernel_spec kernel,
                                rpc_run_config cfg, rpc_result** out) {
  if (cfg.block_size < 1) return fail(ctx, RPC_EINVAL, "block_rpcholesky: block size must be >= 1");
  return run_algo(ctx, x_dev, true, n, d, ldx, layout, kernel, cfg, kAlgoBlock, out);
}

static rpc_run_config simple_cfg(int64_t k, uint64_t seed, uint32_t flags) {
  rpc_run_config c{};
  c.block_size = 1;
  c.mode = RPC_UNTIL_RANK;
  c.target_rank = k;
  c.seed = seed;
  c.stop_tol = 0.0;
  c.flags = flags;
  return c;
}

int rpc_simple_rpcholesky(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                          int layout, rpc_kernel_spec kernel, int64_t k, uint64_t seed,
                          uint32_t flags, rpc_result** out) {
  if (k < 1 || k > n) return fail(ctx, RPC_EINVAL, "simple_rpcholesky: need 1 <= k <= N");
  return run_algo(ctx, x, false, n, d, ldx, layout, kernel, simple_cfg(k, seed, flags),
                  kAlgoSimple, out);
}

int rpc_simple_rpcholesky_device(rpc_ctx* ctx, const double* x_dev, int64_t n, int64_t d,
                                 int64_t ldx, int layout, rpc_kernel_spec kernel, int64_t k,
                                 uint64_t seed, uint32_t flags, rpc_result** out) {
  if (k < 1 || k > n) return fail(ctx, RPC_EINVAL, "simple_rpcholesky: need 1 <= k <= N");
  return run_algo(ctx, x_dev, true, n, d, ldx, layout, kernel, simple_cfg(k, seed, flags),
                  kAlgoSimple, out);
}

int rpc_accelerated_rpcholesky_into(rpc_ctx* ctx, const double* x, int64_t n, int64_t d,
                                    int64_t ldx, int layout, rpc_kernel_spec kernel,
                                    rpc_run_config cfg, double* factor_out, int64_t ld_out,
                                    int64_t cols_out, rpc_result** out) {
  if (!ctx || !out || !factor_out) return fail(ctx, RPC_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  *out = nullptr;
  rpc_result* r = new_result();
  double* reg_ptr = nullptr;
  int rc = guarded(ctx, [&] {
    if (!x && n > 0) raise(RPC_EINVAL, "null point matrix");
    if (ldx < (layout == RPC_ROW_MAJOR ? d : n)) raise(RPC_EINVAL, "leading dimension too small");
    CK(cudaSetDevice(ctx->device));
    // page-lock the caller's buffer for the duration (asynchronous D2H), unless it is already
    // rows [r0, r1) of every column belong to this process (global row indexing)
    const Layout Lz = make_layout(std::max<int64_t>(n, 1), ctx->nshards());
    const int64_t r0 = Lz.row0(ctx->first_shard());
    const int64_t r1 = std::min<int64_t>(n, Lz.row0(ctx->first_shard()) +
                                                (int64_t)ctx->nvirt * Lz.cpr * kChunk);
    if (cols_out < 1 || ld_out < r1 - r0) raise(RPC_EINVAL, "factor buffer too small");
    double* lo = factor_out + r0;
    const size_t span = sizeof(double) * (size_t)((cols_out - 1) * ld_out + (r1 - r0));
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, lo) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned && span > 0) {
      CK(cudaHostRegister(lo, span, cudaHostRegisterPortable));
      reg_ptr = lo;
    }
    HostSink sink;
    sink.p = factor_out;
    sink.ld = ld_out;
    sink.cols = cols_out;
    run_factorization(ctx, x, false, n, d, ldx, layout, kernel, cfg, r, false, kAlgoAccelerated,
                      sink);
  });
  if (reg_ptr) cudaHostUnregister(reg_ptr);
  if (rc) {
    delete r;
    return rc;
  }
  *out = r;
  return RPC_OK;
}

int rpc_result_is_lowmem(const rpc_result* r) { return r ? (int)r->lowmem : 0; }

int64_t rpc_result_n(const rpc_result* r) { return r ? r->n : 0; }
int64_t rpc_result_rank(const rpc_result* r) { return r ? r->kcur : 0; }
int64_t rpc_result_num_rounds(const rpc_result* r) { return r ? (int64_t)r->proposed.size() : 0; }
int64_t rpc_result_block_size(const rpc_result* r) { return r ? r->b : 0; }
int rpc_result_rank_exhausted(const rpc_result* r) { return r ? (int)r->exhausted : 0; }
int64_t rpc_result_surplus(const rpc_result* r) { return r ? r->surplus : 0; }
double rpc_result_captured_sq(const rpc_result* r) { return r ? r->captured_sq : 0.0; }

double rpc_result_relative_trace_error(const rpc_result* r) {
  if (!r || r->n <= 0) return 1.0;
  const double tr = (double)r->n;
  return std::clamp((tr - r->fro2) / tr, 0.0, 1.0);
}

int rpc_result_pivots(const rpc_result* r, int64_t* out) {
  if (!r || (!out && r->kcur)) return RPC_EINVAL;
  std::copy(r->pivots.begin(), r->pivots.end(), out);
  return RPC_OK;
}

int rpc_result_chol_copy(const rpc_result* r, double* out) {
  if (!r || (!out && r->kcur)) return RPC_EINVAL;
  if (r->kcur == 0) return RPC_OK;
  rpc_ctx* ctx = r->ctx;
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(out, r->chol_dev.p, sizeof(double) * r->kcur * r->kcur,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int rpc_result_round(const rpc_result* r, int64_t round, int64_t* proposed, int64_t* accepted,
                     int64_t* n_accepted) {
  if (!r || round < 0 || round >= (int64_t)r->proposed.size()) return RPC_ERANGE;
  if (proposed) std::copy(r->proposed[round].begin(), r->proposed[round].end(), proposed);
  if (accepted) std::copy(r->accepted[round].begin(), r->accepted[round].end(), accepted);
  if (n_accepted) *n_accepted = (int64_t)r->accepted[round].size();
  return RPC_OK;
}

int rpc_result_factor_copy(const rpc_result* r, double* out, int64_t ld, int layout) {
  if (!r) return RPC_EINVAL;
  if (r->lowmem)
    return fail(r->ctx, RPC_EINVAL, "low-memory result: the factor is not stored (LowMemResult)");
  rpc_ctx* ctx = r->ctx;
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t k = r->kcur;
    if (k == 0) return;
    for (const Shard& s : r->shards) {
      if (s.n_loc == 0) continue;
      if (layout == RPC_ROW_MAJOR) {
        if (ld < k) raise(RPC_EINVAL, "leading dimension too small");
        CK(cudaMemcpy2DAsync(out + s.row0 * ld, ld * sizeof(double), s.F.p,
                             r->ldf * sizeof(double), k * sizeof(double), s.n_loc,
                             cudaMemcpyDeviceToHost, st));
      } else {
        if (ld < s.n_loc) raise(RPC_EINVAL, "leading dimension too small");
        // transpose column blocks on the device, then one 2D copy per block
        const int64_t cb = std::max<int64_t>(1, std::min<int64_t>(k, (int64_t)(512ll << 20) / (8 * s.n_loc)));
        DBuf tmp(ctx, sizeof(double) * s.n_loc * cb);
        for (int64_t c0 = 0; c0 < k; c0 += cb) {
          const int64_t nc = std::min(cb, k - c0);
          launch_f_to_colmajor(s.F.as<double>(), r->ldf, s.n_loc, (int)c0, (int)nc,
                               tmp.as<double>(), s.n_loc, st);
          CK(cudaMemcpy2DAsync(out + c0 * ld + s.row0, ld * sizeof(double), tmp.p,
                               s.n_loc * sizeof(double), s.n_loc * sizeof(double), nc,
                               cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
      }
    }
    CK(cudaStreamSynchronize(st));
  });
}

int rpc_result_residual_diag_copy(const rpc_result* r, double* out) {
  if (!r) return RPC_EINVAL;
  rpc_ctx* ctx = r->ctx;
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    for (const Shard& s : r->shards)
      if (s.n_loc)
        CK(cudaMemcpyAsync(out + s.row0, s.u.p, sizeof(double) * s.n_loc, cudaMemcpyDeviceToHost,
                           ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

const double* rpc_result_factor_device(const rpc_result* r, int64_t* ldf, int64_t* row0,
                                       int64_t* nrows) {
  if (!r || r->shards.empty() || r->lowmem) return nullptr;
  if (ldf) *ldf = r->ldf;
  if (row0) *row0 = r->shards[0].row0;
  if (nrows) *nrows = r->shards[0].n_loc;
  return r->shards[0].F.as<double>();
}

int rpc_result_timing(const rpc_result* r, rpc_timing* t) {
  if (!r || !t) return RPC_EINVAL;
  *t = r->timing;
  return RPC_OK;
}

void rpc_result_free(rpc_result* r) {
  if (!r) return;
  if (r->ctx) {
    std::lock_guard<std::mutex> lk(r->ctx->mu);
    cudaStreamSynchronize(r->ctx->stream);
    cudaStreamSynchronize(r->ctx->copy_stream);
    if (r->ctx->aux_stream) cudaStreamSynchronize(r->ctx->aux_stream);
    r->shards.clear();  // buffers return to the ctx pool
    r->chol_dev.release();
  }
  delete r;
}

// ---- bench_column_throughput (experiment.hpp:344-387) ------------------------------
namespace rpcb_rt {
// prop[j] = record of column point cols[j] = SplitMix64(seed) draw (draw0 + j) mod n
__global__ void draw_column_records_kernel(const double* __restrict__ X, const double* __restrict__ sqn,
                                           int64_t n, int64_t dpad, uint64_t seed, uint64_t draw0,
                                           RecordLayout lay, double* __restrict__ prop) {
  const int j = blockIdx.x;
  const int64_t c = (int64_t)(splitmix64_draw(seed, draw0 + (uint64_t)j) % (uint64_t)n);
  double* rec = prop + (int64_t)j * lay.rec;
  if (threadIdx.x == 0) {
    rec[0] = (double)c;
    rec[1] = sqn[c];
  }
  for (int64_t i = threadIdx.x; i < dpad; i += blockDim.x) rec[lay.xoff + i] = X[c * dpad + i];
}
}  // namespace rpcb_rt

// ---- component entry points --------------------------------------------------
// Standalone Gaussian Gram columns go to the tensor-core kernel (i8cols.cu) for d <= 32
// unless RPC_NO_I8COLS is set (the FP64 DMMA columns-only update kernel otherwise).
static bool use_i8cols(int kind, int64_t d, int64_t n) {
  return kind == kGaussGram && d <= kI8ColsMaxD && n < ((int64_t)1 << 31) &&
         !std::getenv("RPC_NO_I8COLS");
}
struct I8ColsBufs {
  DBuf planes, xexp, bplanes, cinfo;
  I8ColsBufs(rpc_ctx* ctx, int64_t n)
      : planes(ctx, i8cols_plane_bytes(n)), xexp(ctx, sizeof(int) * n),
        bplanes(ctx, (size_t)kI8ColsSlices * 128 * 32), cinfo(ctx, sizeof(double) * 384) {}
};

int rpc_bench_column_throughput(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                                int layout, rpc_kernel_spec kspec, const int64_t* block_sizes,
                                int n_sizes, uint64_t seed, rpc_throughput_row* rows,
                                int* n_rows) {
  if (!ctx) return fail(nullptr, RPC_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded(ctx, [&] {
    int kind0 = 0;
    rpc_run_config cfg{1, RPC_UNTIL_RANK, 0, 1, 0, 0.0, 0};
    validate(n, d, kspec, cfg, kind0);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t dpad = round_up(d, 16);
    DBuf X(ctx, sizeof(double) * n * dpad), sqn(ctx, sizeof(double) * n),
        raw(ctx, sizeof(double) * n * d);
    h2d_points(raw.p, x, n, d, ldx, layout, st);
    launch_pack_points(raw.as<double>(), n, (int)d, layout == RPC_ROW_MAJOR ? d : n,
                       layout == RPC_ROW_MAJOR, dpad, X.as<double>(), sqn.as<double>(), nullptr, st);
    RecordLayout lay{2 + dpad, 2, 2 + dpad};
    // Gaussian: Direct and GramTrick (is_l2_translation_invariant); l1: Direct only
    std::vector<int> modes{RPC_DIST_DIRECT};
    if (kspec.kind != RPC_KERNEL_L1LAPLACE) modes.push_back(RPC_DIST_GRAM);
    int64_t maxb = 1;
    for (int i = 0; i < n_sizes; ++i) {
      if (block_sizes[i] < 1) raise(RPC_EINVAL, "bench_column_throughput: block size must be >= 1");
      maxb = std::max(maxb, block_sizes[i]);
    }
    const int64_t mb = std::min<int64_t>(maxb, 256);
    DBuf prop(ctx, sizeof(double) * 256 * lay.rec), pos(ctx, sizeof(int) * 256),
        outd(ctx, sizeof(double) * n * mb), tile(ctx, sizeof(double) * (n / 64 + 2)),
        xs(ctx, sizeof(double) * 256 * dpad), fs(ctx, sizeof(double) * 256 * 16),
        sqnS(ctx, sizeof(double) * 256), idS(ctx, sizeof(double) * 256);
    std::vector<int> hpos(256);
    for (int i = 0; i < 256; ++i) hpos[i] = i;
    CK(cudaMemcpyAsync(pos.p, hpos.data(), sizeof(int) * 256, cudaMemcpyHostToDevice, st));
    // point digit planes for the tensor-core Gram columns: prepared with the points (as the
    // packed copy and the squared norms), outside the timed blocks
    std::unique_ptr<I8ColsBufs> i8b;
    if (kspec.kind != RPC_KERNEL_L1LAPLACE && use_i8cols(kGaussGram, d, n)) {
      i8b.reset(new I8ColsBufs(ctx, n));
      launch_i8cols_prep(X.as<double>(), dpad, (int)d, n, i8b->planes.as<int8_t>(),
                         i8b->xexp.as<int>(), st);
    }
    int nr = 0;
    for (int i = 0; i < n_sizes; ++i) {
      const int64_t b = block_sizes[i];
      for (int mode : modes) {
        rpc_kernel_spec ks = kspec;
        ks.distance_mode = mode;
        int kind = 0;
        validate(n, d, ks, cfg, kind);
        const int64_t n_blocks = (1000 + b - 1) / b;
        auto run = [&]() {
          for (int64_t blk = 0; blk < n_blocks; ++blk) {
            // one oracle.columns(cols) call: b columns, in launches of <= 256
            const int64_t step = (i8b && kind == kGaussGram) ? 128 : 256;
            for (int64_t c0 = 0; c0 < b; c0 += step) {
              const int nc = (int)std::min<int64_t>(step, b - c0);
              draw_column_records_kernel<<<nc, 64, 0, st>>>(X.as<double>(), sqn.as<double>(), n,
                                                             dpad, seed, (uint64_t)(blk * b + c0),
                                                             lay, prop.as<double>());
              if (i8b && kind == kGaussGram && nc >= kI8ColsMinM) {
                double esc = 0.0;
                const int kf = kernel_fun(ks, &esc);
                if (launch_i8cols(i8b->planes.as<int8_t>(), i8b->xexp.as<int>(), sqn.as<double>(),
                                  n, prop.as<double>(), lay.rec, nc, kf, esc,
                                  i8b->bplanes.as<int8_t>(), i8b->cinfo.as<double>(),
                                  outd.as<double>() + (c0 % mb) * n, n, st) < 0)
                  raise(RPC_ECUDA, "tensor-core kernel-column launch failed");
                continue;
              }
              launch_gather_accepted(prop.as<double>(), lay, pos.as<int>(), nc, 256, 0, (int)dpad,
                                     xs.as<double>(), fs.as<double>(), 16, sqnS.as<double>(),
                                     idS.as<double>(), st, nullptr, gram_xscale(kind));
              UpdateParams up{};
              up.X = X.as<double>();
              up.dpad = dpad;
              up.dchunks = (int)(dpad / 16);
        up.d = (int)d;
              up.sqn = sqn.as<double>();
              up.F = X.as<double>();
              up.ldf = dpad;
              up.n_loc = n;
              up.xs = xs.as<double>();
              up.fs = fs.as<double>();
              up.ldfs = 16;
              up.sqnS = sqnS.as<double>();
              up.idS = idS.as<double>();
              up.m = nc;
              up.linv = xs.as<double>();
              up.ldl = 16;
              up.sigma = ks.sigma;
              up.kind = kind;
              up.kfun = kernel_fun(ks, &up.escale);
              up.tile_g2 = tile.as<double>();
              up.columns_only = 1;
              up.cols_out = outd.as<double>() + (c0 % mb) * n;
              up.ld_out = n;
              if (launch_update(up, st) < 0) raise(RPC_ECUDA, "kernel-column launch failed");
            }
          }
        };
        run();  // warm-up (module load, TMA descriptors)
        Ev e0, e1;
        CK(cudaEventRecord(e0.e, st));
        run();
        CK(cudaEventRecord(e1.e, st));
        CK(cudaEventSynchronize(e1.e));
        CK(cudaGetLastError());
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0.e, e1.e));
        rpc_throughput_row& r = rows[nr++];
        r.block_size = b;
        r.distance_mode = mode;
        r.columns = n_blocks * b;
        r.wall_ms = ms;
        r.columns_per_sec = ms > 0 ? 1000.0 * (double)r.columns / ms : 0.0;
        r.output_gbs = ms > 0 ? 8.0 * (double)n * (double)r.columns / (ms * 1e-3) / 1e9 : 0.0;
      }
    }
    *n_rows = nr;
  });
}

int rpc_kernel_columns(rpc_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                       int layout, rpc_kernel_spec kspec, const int64_t* cols, int64_t m,
                       double* out, int64_t ld_out, double* device_ms) {
  if (!ctx) return fail(nullptr, RPC_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded(ctx, [&] {
    int kind = 0;
    rpc_run_config cfg{1, RPC_UNTIL_RANK, 0, 1, 0, 0.0, 0};
    validate(n, d, kspec, cfg, kind);
    for (int64_t j = 0; j < m; ++j)
      if (cols[j] < 0 || cols[j] >= n) raise(RPC_ERANGE, "KernelOracle cols: index out of range");
    if (ld_out < n) raise(RPC_EINVAL, "leading dimension too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t dpad = round_up(d, 16);
    DBuf X(ctx, sizeof(double) * n * dpad), sqn(ctx, sizeof(double) * n),
        raw(ctx, sizeof(double) * n * d);
    h2d_points(raw.p, x, n, d, ldx, layout, st);
    launch_pack_points(raw.as<double>(), n, (int)d, layout == RPC_ROW_MAJOR ? d : n,
                       layout == RPC_ROW_MAJOR, dpad, X.as<double>(), sqn.as<double>(), nullptr,
                       st);
    RecordLayout lay{2 + dpad, 2, 2 + dpad};
    std::unique_ptr<I8ColsBufs> i8b;
    if (use_i8cols(kind, d, n)) {
      i8b.reset(new I8ColsBufs(ctx, n));
      launch_i8cols_prep(X.as<double>(), dpad, (int)d, n, i8b->planes.as<int8_t>(),
                         i8b->xexp.as<int>(), st);
    }
    const int64_t mb = std::min<int64_t>(m, i8b ? 128 : 256);
    DBuf prop(ctx, sizeof(double) * 256 * lay.rec), pos(ctx, sizeof(int) * 256),
        outd(ctx, sizeof(double) * n * std::max<int64_t>(mb, 1)), tile(ctx, sizeof(double) * (n / 64 + 2)),
        xs(ctx, sizeof(double) * 256 * dpad), fs(ctx, sizeof(double) * 256 * 16),
        sqnS(ctx, sizeof(double) * 256), idS(ctx, sizeof(double) * 256);
    std::vector<int> hpos(256);
    for (int i = 0; i < 256; ++i) hpos[i] = i;
    CK(cudaMemcpyAsync(pos.p, hpos.data(), sizeof(int) * 256, cudaMemcpyHostToDevice, st));
    double total_ms = 0.0;
    Ev e0, e1;
    for (int64_t c0 = 0; c0 < m; c0 += mb) {
      const int64_t nc = std::min(mb, m - c0);
      // records: id, ||x||^2, x (from the packed device copy)
      for (int64_t j = 0; j < nc; ++j) {
        CK(cudaMemcpyAsync(prop.as<double>() + j * lay.rec + 1, sqn.as<double>() + cols[c0 + j],
                           sizeof(double), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(prop.as<double>() + j * lay.rec + 2,
                           X.as<double>() + cols[c0 + j] * dpad, sizeof(double) * dpad,
                           cudaMemcpyDeviceToDevice, st));
      }
      std::vector<double> ids(nc);
      for (int64_t j = 0; j < nc; ++j) ids[j] = (double)cols[c0 + j];
      CK(cudaMemcpy2DAsync(prop.p, lay.rec * 8, ids.data(), 8, 8, nc, cudaMemcpyHostToDevice, st));
      launch_gather_accepted(prop.as<double>(), lay, pos.as<int>(), (int)nc, 256, 0, (int)dpad,
                             xs.as<double>(), fs.as<double>(), 16, sqnS.as<double>(),
                             idS.as<double>(), st, nullptr, gram_xscale(kind));
      UpdateParams up{};
      up.X = X.as<double>();
      up.dpad = dpad;
      up.dchunks = (int)(dpad / 16);
        up.d = (int)d;
      up.sqn = sqn.as<double>();
      up.F = X.as<double>();
      up.ldf = dpad;
      up.kcur = 0;
      up.u = nullptr;
      up.n_loc = n;
      up.row0 = 0;
      up.xs = xs.as<double>();
      up.fs = fs.as<double>();
      up.ldfs = 16;
      up.sqnS = sqnS.as<double>();
      up.idS = idS.as<double>();
      up.m = (int)nc;
      up.linv = xs.as<double>();
      up.ldl = 16;
      up.sigma = kspec.sigma;
      up.kind = kind;
      up.kfun = kernel_fun(kspec, &up.escale);
      up.tile_g2 = tile.as<double>();
      up.columns_only = 1;
      up.cols_out = outd.as<double>();
      up.ld_out = n;
      CK(cudaEventRecord(e0.e, st));
      const int bm =
          (i8b && nc >= kI8ColsMinM) ? launch_i8cols(i8b->planes.as<int8_t>(), i8b->xexp.as<int>(), sqn.as<double>(), n,
                              prop.as<double>(), lay.rec, (int)nc, up.kfun, up.escale,
                              i8b->bplanes.as<int8_t>(), i8b->cinfo.as<double>(),
                              outd.as<double>(), n, st)
              : launch_update(up, st);
      if (bm < 0) raise(RPC_ECUDA, "kernel-column launch failed (code " + std::to_string(bm) + ")");
      CK(cudaEventRecord(e1.e, st));
      CK(cudaMemcpy2DAsync(out + c0 * ld_out, ld_out * 8, outd.p, n * 8, n * 8, nc,
                           cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0.e, e1.e));
      total_ms += ms;
    }
    CK(cudaGetLastError());
    if (device_ms) *device_ms = total_ms;
  });
}

int rpc_sample_discrete(rpc_ctx* ctx, const double* u, int64_t n, int64_t b, uint64_t seed,
                        uint64_t draw0, int replay, int64_t* out) {
  if (!ctx) return fail(nullptr, RPC_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded(ctx, [&] {
    if (n == 0) raise(RPC_EINVAL, "sample_discrete: empty weights");
    if (b < 1 || b > 65535) raise(RPC_EINVAL, "sample_discrete: bad draw count");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const Layout L = make_layout(n, 1);
    DBuf du(ctx, sizeof(double) * n), totals(ctx, sizeof(double) * L.ncg),
        cend(ctx, sizeof(double) * L.ncg), status(ctx, sizeof(ScanStatus)),
        rec(ctx, sizeof(double) * 2 * b), owner(ctx, sizeof(int) * b), c0(ctx, sizeof(int) * 2),
        zeros(ctx, sizeof(double) * n), cs;
    CK(cudaMemcpyAsync(du.p, u, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(zeros.p, 0, sizeof(double) * n, st));
    int hc0[2] = {0, L.ncg};
    CK(cudaMemcpyAsync(c0.p, hc0, sizeof hc0, cudaMemcpyHostToDevice, st));
    SampleParams sp{};
    sp.u = du.as<double>();
    sp.X = zeros.as<double>();
    sp.sqn = zeros.as<double>();
    sp.F = zeros.as<double>();
    sp.n_loc = n;
    sp.n_global = n;
    sp.dpad = 0;
    sp.ldf = 0;
    sp.kcur = 0;
    sp.chunk0 = 0;
    sp.n_chunks_local = L.nc;
    sp.n_chunks_global = L.ncg;
    sp.shard = 0;
    sp.n_shards = 1;
    sp.shard_chunk0 = c0.as<int>();
    sp.chunk_end = cend.as<double>();
    sp.seed = seed;
    sp.draw0 = draw0;
    sp.b = (int)b;
    sp.lay = RecordLayout{2, 2, 2};
    sp.records = rec.as<double>();
    sp.owner = owner.as<int>();
    ScanStatus hs{};
    if (replay) {
      cs = DBuf(ctx, sizeof(double) * n);
      launch_replay_scan(du.as<double>(), n, cs.as<double>(), status.as<ScanStatus>(), st);
      CK(cudaMemcpyAsync(&hs, status.p, sizeof hs, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (hs.exhausted) raise(RPC_EINVAL, "sample_discrete: total weight must be > 0");
      launch_replay_sample(sp, cs.as<double>(), st);
    } else {
      // thread bases for the sampler (RPC_NO_TB_SAMPLER: the rescanning sampler instead)
      DBuf tbd(ctx, sizeof(double) * (size_t)L.ncg * kScanThreads);
      launch_chunk_totals(du.as<double>(), n, L.nc, totals.as<double>(), st, nullptr, 0, nullptr,
                          FusedPrefix(), tbd.as<double>());
      if (!std::getenv("RPC_NO_TB_SAMPLER")) sp.tb = tbd.as<double>();
      CK(cudaMemsetAsync(totals.as<double>() + L.nc, 0, sizeof(double) * (L.ncg - L.nc), st));
      launch_chunk_prefix(totals.as<double>(), nullptr, L.ncg, cend.as<double>(),
                          status.as<ScanStatus>(), st);
      CK(cudaMemcpyAsync(&hs, status.p, sizeof hs, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (hs.exhausted) raise(RPC_EINVAL, "sample_discrete: total weight must be > 0");
      launch_sample(sp, st);
    }
    std::vector<double> h(2 * b);
    CK(cudaMemcpyAsync(h.data(), rec.p, sizeof(double) * 2 * b, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    for (int64_t j = 0; j < b; ++j) out[j] = (int64_t)h[2 * j];
  });
}

int rpc_rejection_sweep(rpc_ctx* ctx, const double* h, int64_t b, const int64_t* proposals,
                        uint64_t seed, uint64_t draw0, int64_t* accepted, int64_t* positions,
                        int64_t* m_out, double* chol) {
  if (!ctx) return fail(nullptr, RPC_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  return guarded(ctx, [&] {
    if (b < 1 || b > kMaxBlock) raise(RPC_EINVAL, "rejection_sample_submatrix: size mismatch");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    std::vector<double> hrm((size_t)b * b), rec((size_t)2 * b);
    for (int64_t p = 0; p < b; ++p)
      for (int64_t q = 0; q < b; ++q) hrm[p * b + q] = h[q * b + p];
    for (int64_t j = 0; j < b; ++j) {
      rec[2 * j] = (double)proposals[j];
      rec[2 * j + 1] = 0.0;
    }
    DBuf dH(ctx, sizeof(double) * b * b), dprop(ctx, sizeof(double) * 2 * b),
        dpos(ctx, sizeof(int) * b), dids(ctx, sizeof(int64_t) * b),
        dl(ctx, sizeof(double) * b * b), dla(ctx, sizeof(double) * b * b),
        dout(ctx, sizeof(SweepOut)), dhp(ctx, sizeof(double) * (b * (b + 1) / 2 + 1));
    CK(cudaMemcpyAsync(dH.p, hrm.data(), sizeof(double) * b * b, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dprop.p, rec.data(), sizeof(double) * 2 * b, cudaMemcpyHostToDevice, st));
    launch_sweep(dH.as<double>(), (int)b, seed, draw0, dprop.as<double>(), RecordLayout{2, 2, 2},
                 dpos.as<int>(), dids.as<int64_t>(), dl.as<double>(), dla.as<double>(),
                 dout.as<SweepOut>(), dhp.as<double>(), st);
    SweepOut so{};
    CK(cudaMemcpyAsync(&so, dout.p, sizeof so, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int m = so.m;
    std::vector<int> hp(m);
    if (m) {
      CK(cudaMemcpyAsync(hp.data(), dpos.p, sizeof(int) * m, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(accepted, dids.p, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(chol, dla.p, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    for (int i = 0; i < m; ++i) positions[i] = hp[i];
    *m_out = m;
  });
}

}  // extern "C"
