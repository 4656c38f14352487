// io.cu — on-disk output contract of the factor (io.hpp:218-293, 336-350) written straight
// from the device-resident result.
//
// RPCF: "RPCF", u32 version 1, u64 N, u64 k, k*N f64 column-major, k u64 pivots, u64 packed
// Cholesky count k(k+1)/2, the lower triangle of chol_factor row by row.  The factor lives
// row-major in HBM, so it is streamed out in column blocks: a transpose kernel writes block
// c into one half of a pinned staging area while the host pwrite()s block c-1 from the
// other half (D2H + file write overlapped).  Each process writes its own row segment of
// every column at its file offset, so a multi-GPU result is written in parallel without a
// gather; rank 0 creates and sizes the file and writes header and trailer.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cinttypes>

#include "runtime.h"

namespace rpcb_rt {
namespace {

__global__ void pack_chol_rows_kernel(const double* __restrict__ chol_cm, int64_t k,
                                      double* __restrict__ packed) {
  const int64_t i = blockIdx.x;  // row i: entries (i, 0..i)
  double* dst = packed + i * (i + 1) / 2;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) dst[j] = chol_cm[j * k + i];
}

void pwrite_all(int fd, const void* buf, size_t bytes, off_t off, const char* path) {
  const char* p = static_cast<const char*>(buf);
  while (bytes > 0) {
    const ssize_t w = pwrite(fd, p, bytes, off);
    if (w <= 0) raise(RPC_ENUMERIC, std::string("write_rpcf: write failed for ") + path);
    p += w;
    bytes -= (size_t)w;
    off += w;
  }
}

}  // namespace
}  // namespace rpcb_rt

using namespace rpcb_rt;

extern "C" {

int rpc_result_write_rpcf(const rpc_result* r, const char* path) {
  if (!r || !path) return RPC_EINVAL;
  rpc_ctx* ctx = r->ctx;
  if (r->lowmem)
    return fail(ctx, RPC_EINVAL, "write_rpcf: low-memory result has no factor");
  return guarded(ctx, [&] {
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const uint64_t n = (uint64_t)r->n, k = (uint64_t)r->kcur;
    const off_t hdr = 24, f_off = hdr, piv_off = hdr + (off_t)(8 * k * n);
    const off_t cnt_off = piv_off + (off_t)(8 * k), chol_off = cnt_off + 8;
    const uint64_t chol_count = k > 0 ? k * (k + 1) / 2 : 0;
    const off_t total = chol_off + (off_t)(8 * chol_count);
    const bool lead = ctx->rank == 0;
    DBuf tok(ctx, sizeof(uint64_t));
    struct Closer {
      int fd = -1;
      ~Closer() {
        if (fd >= 0) close(fd);
      }
    } closer;
    // rank 0 creates and sizes the file; every rank learns whether that worked before any
    // rank writes (so a failure raises everywhere instead of leaving ranks in a collective)
    bool bad = false;
    if (lead) {
      closer.fd = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
      bad = closer.fd < 0 || ftruncate(closer.fd, total) != 0;
    }
    if (any_rank(ctx, bad, tok.p))
      raise(RPC_ENUMERIC, std::string("cannot open for writing: ") + path);
    if (!lead) {
      closer.fd = open(path, O_WRONLY);
      bad = closer.fd < 0;
    }
    if (any_rank(ctx, bad, tok.p))
      raise(RPC_ENUMERIC, std::string("cannot open for writing: ") + path);
    const int fd = closer.fd;
    // every rank writes its rows; a failure on any rank is raised on all of them after the
    // closing barrier, so no rank returns while another is still writing or is left waiting
    RpcError err{RPC_OK, ""};
    try {
      if (lead) {
        char h[24];
        std::memcpy(h, "RPCF", 4);
        const uint32_t ver = 1;
        std::memcpy(h + 4, &ver, 4);  // little-endian host (x86-64)
        std::memcpy(h + 8, &n, 8);
        std::memcpy(h + 16, &k, 8);
        pwrite_all(fd, h, 24, 0, path);
      }
      // ---- factor: column blocks, transpose on the device, double-buffered D2H + pwrite ----
      const size_t half = (size_t)256 << 20;
      if (ctx->io_pinned_bytes < 2 * half) {
        if (ctx->io_pinned) cudaFreeHost(ctx->io_pinned);
        ctx->io_pinned = nullptr;
        CK(cudaMallocHost(&ctx->io_pinned, 2 * half));
        ctx->io_pinned_bytes = 2 * half;
      }
      char* stage[2] = {static_cast<char*>(ctx->io_pinned), static_cast<char*>(ctx->io_pinned) + half};
      DBuf dtmp[2] = {DBuf(ctx, half), DBuf(ctx, half)};
      Ev evs[2];
      cudaEvent_t ev[2] = {evs[0].e, evs[1].e};
      struct Pending {
        int buf;
        int64_t c0, nc, row0, nrows;
      };
      std::vector<Pending> pend;
      auto flush = [&](const Pending& q) {
        CK(cudaEventSynchronize(ev[q.buf]));
        for (int64_t c = 0; c < q.nc; ++c)
          pwrite_all(fd, stage[q.buf] + (size_t)(c * q.nrows) * 8, (size_t)q.nrows * 8,
                     f_off + (off_t)(8 * ((uint64_t)(q.c0 + c) * n + (uint64_t)q.row0)), path);
      };
      int buf = 0;
      for (const Shard& s : r->shards) {
        if (s.n_loc == 0 || k == 0) continue;
        const int64_t cb = std::max<int64_t>(1, std::min<int64_t>((int64_t)k, (int64_t)(half / (8 * s.n_loc))));
        if ((size_t)s.n_loc * 8 > half) raise(RPC_EINVAL, "write_rpcf: shard too tall for the staging buffer");
        for (int64_t c0 = 0; c0 < (int64_t)k; c0 += cb) {
          const int64_t nc = std::min<int64_t>(cb, (int64_t)k - c0);
          // the staging half about to be reused must have been written out
          if (pend.size() >= 2) {
            flush(pend.front());
            pend.erase(pend.begin());
          }
          launch_f_to_colmajor(s.F.as<double>(), r->ldf, s.n_loc, (int)c0, (int)nc,
                               dtmp[buf].as<double>(), s.n_loc, st);
          CK(cudaMemcpyAsync(stage[buf], dtmp[buf].p, (size_t)(nc * s.n_loc) * 8,
                             cudaMemcpyDeviceToHost, st));
          CK(cudaEventRecord(ev[buf], st));
          pend.push_back({buf, c0, nc, s.row0, s.n_loc});
          buf ^= 1;
          if (pend.size() == 2) {  // overlap: write the older block while this one copies
            flush(pend.front());
            pend.erase(pend.begin());
          }
        }
      }
      for (const Pending& q : pend) flush(q);
      // ---- trailer: pivots, packed Cholesky rows (rank 0) ----
      if (lead) {
        std::vector<uint64_t> piv(r->pivots.begin(), r->pivots.end());
        if (k) pwrite_all(fd, piv.data(), 8 * k, piv_off, path);
        pwrite_all(fd, &chol_count, 8, cnt_off, path);
        if (chol_count) {
          DBuf packed(ctx, sizeof(double) * chol_count);
          pack_chol_rows_kernel<<<(unsigned)k, 128, 0, st>>>(r->chol_dev.as<double>(), (int64_t)k,
                                                             packed.as<double>());
          std::vector<double> h(chol_count);
          CK(cudaMemcpyAsync(h.data(), packed.p, 8 * chol_count, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          pwrite_all(fd, h.data(), 8 * chol_count, chol_off, path);
        }
      }
      CK(cudaStreamSynchronize(st));
    } catch (const RpcError& e) {
      err = e;
    }
    if (any_rank(ctx, err.code != RPC_OK, tok.p))
      raise(err.code != RPC_OK ? err.code : RPC_ENUMERIC,
            err.code != RPC_OK ? err.msg : std::string("write_rpcf: failed on another rank: ") + path);
    CK(cudaStreamSynchronize(st));
  });
}

// write_pivot_trace_csv (io.hpp:336-350): round,proposed,accepted,acceptance_rate (%.17g)
int rpc_result_write_trace_csv(const rpc_result* r, const char* path) {
  if (!r || !path) return RPC_EINVAL;
  return guarded(r->ctx, [&] {
    FILE* f = std::fopen(path, "w");
    if (!f) raise(RPC_ENUMERIC, std::string("cannot open for writing: ") + path);
    std::fprintf(f, "round,proposed,accepted,acceptance_rate\n");
    for (size_t i = 0; i < r->proposed.size(); ++i) {
      const size_t np = r->proposed[i].size(), na = r->accepted[i].size();
      const double rate = np ? (double)na / (double)np : 0.0;
      std::fprintf(f, "%zu,%zu,%zu,%.17g\n", i, np, na, rate);
    }
    std::fclose(f);
  });
}

}  // extern "C"
