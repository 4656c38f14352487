// runtime.h — host runtime shared by the C-ABI translation units (internal):
// error handling, the device context (stream, pool allocator, NCCL comm), device
// buffers, the row-shard layout and the factorization result handle.
#pragma once
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rpchol_gpu.h"
#include "common.cuh"
#include "kernels.h"

using namespace rpcb;

namespace rpcb_rt {

struct RpcError {
  int code;
  std::string msg;
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw RpcError{code, msg}; }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(e == cudaErrorMemoryAllocation ? RPC_ENOMEM : RPC_ECUDA,
          std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) cuda_check((x), #x)

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) raise(RPC_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define NK(x) nccl_check((x), #x)

inline thread_local std::string g_last_error;

// RPC_DEBUG_SYNC=1: synchronise and check after every launch (localises faults).
inline bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("RPC_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
inline void dbg(cudaStream_t st, const char* what) {
  if (!debug_sync()) return;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw RpcError{RPC_ECUDA, std::string("after ") + what + ": " + cudaGetErrorString(e)};
  }
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// NVTX range for profilers (header-only NVTX v3; a no-op unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace rpcb_rt
using namespace rpcb_rt;

struct rpc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // factor streaming to the host (overlaps the rounds)
  cudaStream_t aux_stream = nullptr;   // digit-plane appends beside the next round's chain
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  bool hostcoll = false;      // collectives through caller-provided host callbacks
  rpc_host_collectives hc{};
  void* hc_pinned = nullptr;  // staging for host collectives (send | recv)
  size_t hc_pinned_bytes = 0;
  int nvirt = 1;
  std::mutex mu;
  std::string err;
  std::multimap<size_t, void*> pool;  // cached device blocks (size -> ptr)
  void* host_pinned = nullptr;
  size_t host_pinned_bytes = 0;
  void* io_pinned = nullptr;  // RPCF writer staging (2 halves), grown on demand
  size_t io_pinned_bytes = 0;
  std::vector<void (*)(rpc_ctx*)> on_destroy;

  int nshards() const { return world * nvirt; }
  int first_shard() const { return rank * nvirt; }

  void* dalloc(size_t bytes) {
    bytes = std::max<size_t>(256, round_up((int64_t)bytes, 256));
    auto it = pool.lower_bound(bytes);
    if (it != pool.end() && it->first <= bytes * 2) {
      void* p = it->second;
      pool.erase(it);
      return p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {  // release the cache and retry once
      cudaGetLastError();
      trim();
      CK(cudaMalloc(&p, bytes));
    }
    return p;
  }
  void dfree(void* p, size_t bytes) {
    if (!p) return;
    bytes = std::max<size_t>(256, round_up((int64_t)bytes, 256));
    pool.emplace(bytes, p);
  }
  void trim() {
    cudaStreamSynchronize(stream);
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    if (aux_stream) cudaStreamSynchronize(aux_stream);
    for (auto& kv : pool) cudaFree(kv.second);
    pool.clear();
  }
  void* pinned(size_t bytes) {
    if (bytes > host_pinned_bytes) {
      if (host_pinned) cudaFreeHost(host_pinned);
      host_pinned = nullptr;
      CK(cudaMallocHost(&host_pinned, bytes));
      host_pinned_bytes = bytes;
    }
    return host_pinned;
  }
};

namespace rpcb_rt {

// Device buffer owned through the ctx pool.
struct DBuf {
  rpc_ctx* ctx = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(rpc_ctx* c, size_t b) : ctx(c), bytes(b) { p = b ? c->dalloc(b) : nullptr; }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    ctx = o.ctx;
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p && ctx) ctx->dfree(p, bytes);
    p = nullptr;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Layout {
  int64_t n = 0;
  int P = 1;
  int nc = 0;    // real chunks
  int cpr = 0;   // chunks per shard
  int ncg = 0;   // P * cpr
  int64_t row0(int s) const { return std::min<int64_t>(n, (int64_t)s * cpr * kChunk); }
  int64_t rows(int s) const {
    return std::min<int64_t>(n, (int64_t)(s + 1) * cpr * kChunk) - row0(s);
  }
  int chunks(int s) const { return (int)((rows(s) + kChunk - 1) / kChunk); }
};

inline Layout make_layout(int64_t n, int P) {
  Layout L;
  L.n = n;
  L.P = P;
  L.nc = (int)((n + kChunk - 1) / kChunk);
  L.cpr = (L.nc + P - 1) / P;
  L.ncg = L.cpr * P;
  return L;
}

struct Shard {
  int gidx = 0;  // global shard index
  int64_t row0 = 0, n_loc = 0;
  int chunk0 = 0, nchunks = 0;
  DBuf X, sqn, F, u, tile_g2;
};

}  // namespace rpcb_rt

struct rpc_result {
  rpc_ctx* ctx = nullptr;
  int64_t n = 0, d = 0, kcur = 0, ldf = 0, b = 0;
  std::vector<Shard> shards;
  std::vector<int64_t> pivots;
  std::vector<std::vector<int64_t>> proposed, accepted;
  bool exhausted = false;
  bool lowmem = false;       // accelerated_rpcholesky_lowmem: no factor is kept
  int64_t surplus = 0;
  double captured_sq = 0.0;
  double fro2 = 0.0;
  DBuf chol_dev;             // kcur x kcur column-major lower triangle (device)
  rpc_timing timing{};
};

namespace rpcb_rt {

inline int fail(rpc_ctx* ctx, int code, const std::string& msg) {
  g_last_error = msg;
  if (ctx) ctx->err = msg;
  return code;
}

template <class F>
inline int guarded(rpc_ctx* ctx, F&& f) {
  try {
    f();
    return RPC_OK;
  } catch (const RpcError& e) {
    return fail(ctx, e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return fail(ctx, RPC_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return fail(ctx, RPC_ENUMERIC, e.what());
  }
}

// ---- collectives across the ranks of a context ------------------------------------
// Two are needed: an in-place allgather of per-shard slots (chunk totals,
// ||G||^2 partials, the replay-mode residual diagonal) and an in-place "owner" reduce, where
// at most one rank holds a non-zero word per position (proposal records, chol rows, flags):
// NCCL reduces the bit patterns as uint64 with max, which returns the owner's word bit for
// bit (signed zeros and NaN payloads included).  World 1 (virtual shards) needs neither.
inline void* hc_staging(rpc_ctx* ctx, size_t bytes) {
  if (bytes > ctx->hc_pinned_bytes) {
    if (ctx->hc_pinned) cudaFreeHost(ctx->hc_pinned);
    ctx->hc_pinned = nullptr;
    ctx->hc_pinned_bytes = 0;
    CK(cudaMallocHost(&ctx->hc_pinned, bytes));
    ctx->hc_pinned_bytes = bytes;
  }
  return ctx->hc_pinned;
}

// Allgather of `count` doubles per global shard, in place in buf[P][count].
inline void allgather(rpc_ctx* ctx, double* buf, size_t count) {
  if (ctx->world == 1) return;  // virtual shards already write into buf directly
  const size_t mine = count * ctx->nvirt, off = (size_t)ctx->rank * mine;
  if (!ctx->hostcoll) {
    NK(ncclAllGather(buf + off, buf, mine, ncclDouble, ctx->comm, ctx->stream));
    return;
  }
  const size_t bytes = sizeof(double) * mine;
  char* h = static_cast<char*>(hc_staging(ctx, bytes * (1 + ctx->world)));
  CK(cudaMemcpyAsync(h, buf + off, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->hc.allgather(ctx->hc.user, h, h + bytes, bytes) != 0)
    raise(RPC_ENCCL, "host collective allgather failed");
  CK(cudaMemcpyAsync(buf, h + bytes, bytes * ctx->world, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // h is reused by the next collective
}

// In-place owner reduce of `words` 64-bit words (see above).
inline void allreduce_owner(rpc_ctx* ctx, void* buf, size_t words) {
  if (ctx->world == 1 || words == 0) return;
  if (!ctx->hostcoll) {
    NK(ncclAllReduce(buf, buf, words, ncclUint64, ncclMax, ctx->comm, ctx->stream));
    return;
  }
  const size_t bytes = sizeof(uint64_t) * words;
  uint64_t* h = static_cast<uint64_t*>(hc_staging(ctx, bytes));
  CK(cudaMemcpyAsync(h, buf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->hc.allreduce_or_u64(ctx->hc.user, h, words) != 0)
    raise(RPC_ENCCL, "host collective allreduce failed");
  CK(cudaMemcpyAsync(buf, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // h is reused by the next collective
}

// Host flag agreed by every rank (OR): lets all ranks raise together instead of leaving
// the others blocked in the next collective.  `scratch` is an 8-byte device word.
inline bool any_rank(rpc_ctx* ctx, bool flag, void* scratch) {
  if (ctx->world == 1) return flag;
  uint64_t v = flag ? 1 : 0;
  CK(cudaMemcpyAsync(scratch, &v, sizeof v, cudaMemcpyHostToDevice, ctx->stream));
  allreduce_owner(ctx, scratch, 1);
  CK(cudaMemcpyAsync(&v, scratch, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return v != 0;
}

inline void validate(int64_t n, int64_t d, const rpc_kernel_spec& k, rpc_run_config& cfg, int& kind) {
  if (n < 1 || d < 1) raise(RPC_EINVAL, "DataMatrix: need at least one point and one dimension");
  if (!(k.sigma > 0.0) || !std::isfinite(k.sigma))
    raise(RPC_EINVAL, "KernelSpec: bandwidth must be positive");
  int mode = k.distance_mode;
  if (k.kind == RPC_KERNEL_GAUSSIAN || k.kind == RPC_KERNEL_MATERN32 ||
      k.kind == RPC_KERNEL_MATERN52) {  // l2 translation-invariant (kernels.hpp:55-57)
    if (mode == RPC_DIST_DEFAULT) mode = RPC_DIST_GRAM;
    if (mode != RPC_DIST_GRAM && mode != RPC_DIST_DIRECT) raise(RPC_EINVAL, "unknown distance mode");
    kind = mode == RPC_DIST_GRAM ? kGaussGram : kGaussDirect;
  } else if (k.kind == RPC_KERNEL_L1LAPLACE) {
    if (mode == RPC_DIST_DEFAULT) mode = RPC_DIST_DIRECT;
    if (mode == RPC_DIST_GRAM)
      raise(RPC_EINVAL, "KernelOracle: GramTrick requires an l2 translation-invariant kernel");
    kind = kL1;
  } else {
    raise(RPC_EINVAL, "unknown kernel kind");
  }
  if (cfg.block_size < 1) raise(RPC_EINVAL, "accelerated_rpcholesky: block size must be >= 1");
  if (cfg.block_size > kMaxBlock)
    raise(RPC_EINVAL, "accelerated_rpcholesky: this build supports block size <= " +
                          std::to_string(kMaxBlock));
  if (cfg.mode == RPC_FIXED_ROUNDS) {
    if (cfg.rounds < 1) raise(RPC_EINVAL, "RunConfig: t, b must be >= 1");
  } else if (cfg.mode == RPC_UNTIL_RANK) {
    if (cfg.target_rank < 1) raise(RPC_EINVAL, "RunConfig: k, b must be >= 1");
  } else {
    raise(RPC_EINVAL, "RunConfig: unknown mode");
  }
}

// KernelFun id and its scale for the device transforms (kernels.hpp:60-79; l1: oracle.hpp:303).
inline int kernel_fun(const rpc_kernel_spec& k, double* scale) {
  const double sg = k.sigma;
  switch (k.kind) {
    case RPC_KERNEL_MATERN32: *scale = 1.0 / sg; return kFunMatern32;
    case RPC_KERNEL_MATERN52: *scale = 1.0 / (sg * sg); return kFunMatern52;
    case RPC_KERNEL_L1LAPLACE: *scale = -1.0 / sg; return kFunExp;
    default: *scale = -0.5 / (sg * sg); return kFunExp;
  }
}

struct Ev {
  cudaEvent_t e = nullptr;
  Ev() { CK(cudaEventCreate(&e)); }
  Ev(const Ev&) = delete;
  Ev& operator=(const Ev&) = delete;
  Ev(Ev&& o) noexcept : e(o.e) { o.e = nullptr; }
  ~Ev() {
    if (e) cudaEventDestroy(e);
  }
};

// Host points (n x d, either layout, leading dimension ldx) -> dense device copy (row-major
// [n][d] or column-major [d][n] as given).  Contiguous inputs go as one linear copy: a pitched
// copy of 8d-byte rows runs at a few GB/s.
inline void h2d_points(void* dst, const double* x, int64_t n, int64_t d, int64_t ldx, int layout,
                       cudaStream_t st) {
  const int64_t inner = layout == RPC_ROW_MAJOR ? d : n, outer = layout == RPC_ROW_MAJOR ? n : d;
  if (ldx == inner)
    CK(cudaMemcpyAsync(dst, x, sizeof(double) * inner * outer, cudaMemcpyHostToDevice, st));
  else
    CK(cudaMemcpy2DAsync(dst, inner * 8, x, ldx * 8, inner * 8, outer, cudaMemcpyHostToDevice, st));
}

// The factorization proper (api.cu).  `src` points to this process's shard rows
// (device memory when src_on_device, else host memory of the full X).
enum { kAlgoAccelerated = 0, kAlgoBlock = 1, kAlgoSimple = 2 };
// Host destination for the factor, filled while the rounds run: column-major, leading
// dimension ld >= N, at least `cols` columns (this process's rows only).
struct HostSink {
  double* p = nullptr;
  int64_t ld = 0, cols = 0;
};
void run_factorization(rpc_ctx* ctx, const double* src, bool src_on_device, int64_t n,
                       int64_t d, int64_t ldx, int layout, const rpc_kernel_spec& kspec,
                       rpc_run_config cfg, rpc_result* res, bool lowmem = false,
                       int algo = kAlgoAccelerated, HostSink sink = HostSink());

}  // namespace rpcb_rt
