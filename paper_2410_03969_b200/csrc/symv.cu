// symv.cu — symmetric kernel matvec for KRR (kernel_matvec, krr.hpp:143-162, one right-hand
// side, training points against themselves): out = A v + add_coef * add_vec.
//
// A(i, j) = kappa(x_i, x_j) is symmetric, so only the lower block triangle is generated:
// the rows and columns are cut into super-blocks of kSB = 1024 points, and each unit
// (I >= J) regenerates the 1024 x 1024 block A(I, J) once and uses it twice,
//   rowpart(I, J) = A(I, J) v(J)        and, for I > J,   colpart(I, J) = A(I, J)^T v(I),
// which halves the kernel evaluations (Gram products on DMMA + exp, or l1 / direct
// distances on the FP64 cores) that dominate the product.  Determinism without atomics:
// a unit is processed by one warp group in a fixed order (row tiles, then 16-column chunks),
// each warp keeps its column partials in its own shared-memory slots, the four warps' slots
// are combined in warp order, and a final pass sums, per output row, the unit partials in
// block order.  Results are bit-reproducible run to run.
//
// Execution follows the low-memory update kernel's single-warp-column path (lowmem_impl.cuh):
// persistent CTAs of two groups of four warps, a row tile's points X(R, :) resident in shared
// memory, the 16 column points of each chunk and the v chunk streamed by TMA through an
// S-stage ring, the 16 x 16 kernel tile of each warp kept in registers.
#include "update_impl.cuh"

namespace rpcb {

namespace {

constexpr int kSB = 1024;          // super-block (points)
constexpr int kRT = kSB / 64;      // row tiles per super-block
constexpr int kCH = kSB / 16;      // column chunks per super-block
constexpr int kNCW = 4;            // warps per group
constexpr int kGT = 32 * kNCW;
constexpr int kG = 2;              // groups per CTA

struct SymvParams {
  const double* X; int64_t dpad; int dchunks; int d;  // points [n][dpad]
  const double* sqn;                                  // ||x||^2
  const double* rec; int64_t prec;                    // records: id, ||x||^2, x
  const double* v;                                    // [n]
  int64_t n;
  int kind; int kfun; double escale;
  int nsb, nunits;
  double* rowpart;                                    // [nunits][kSB]
  double* colpart;                                    // [nunits][kSB]
};

__host__ __device__ inline int stage_bytes(int nD) { return nD * 2048 + 1024; }
__host__ __device__ inline int group_bytes(int S, int nD) {
  return S * stage_bytes(nD) + nD * 64 * 128 + kNCW * kSB * 8;
}
__host__ __device__ inline int smem_bytes(int S, int nD) {
  return kG * group_bytes(S, nD) + 64 * 8 + kG * (2 * 8 + 2 * 8 * 8) + 1024;
}

__device__ __forceinline__ void unit_of(int u, int& I, int& J) {
  I = (int)((sqrtf(8.0f * u + 1.0f) - 1.0f) * 0.5f);
  while (I * (I + 1) / 2 > u) --I;
  while ((I + 1) * (I + 2) / 2 <= u) ++I;
  J = u - I * (I + 1) / 2;
}

template <bool GRAM>
__global__ void __launch_bounds__(256, 2)
    symv_kernel(SymvParams p, int S, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmXS, const __grid_constant__ CUtensorMap tmW) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t align = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = (tid >> 5) / kNCW, warp = (tid >> 5) % kNCW, gtid = tid % kGT;
  const int nD = p.dchunks;
  const int STAGE = stage_bytes(nD);
  unsigned char* gbase = smem_raw + align + grp * group_bytes(S, nD);
  unsigned char* stages = gbase;                                   // [S][XS nD x 2 KB | W 1 KB]
  unsigned char* xt = gbase + S * STAGE;                           // X(R, :) [nD][64][16]
  double* colacc = reinterpret_cast<double*>(xt + nD * 64 * 128);  // [kNCW][kSB]
  double* s_exp2 = reinterpret_cast<double*>(smem_raw + align + kG * group_bytes(S, nD));
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_exp2 + 64) + grp * (2 + 2 * 8);
  uint64_t* xbar = bars;
  uint64_t* full = bars + 2;
  uint64_t* empty = full + 8;
  auto gsync = [&]() { named_bar_sync(1 + grp, kGT); };

  const int vb = (int)blockIdx.x * kG + grp, vgrid = (int)gridDim.x * kG;
  auto unit_dims = [&](int u, int& I, int& J, int& nrt, int& nch) {
    unit_of(u, I, J);
    nrt = (int)min((int64_t)kRT, (p.n - (int64_t)I * kSB + 63) / 64);
    nch = (int)min((int64_t)kCH, (p.n - (int64_t)J * kSB + 15) / 16);
  };
  int total = 0;  // chunks this group consumes
  for (int u = vb; u < p.nunits; u += vgrid) {
    int I, J, nrt, nch;
    unit_dims(u, I, J, nrt, nch);
    total += nrt * nch;
  }
  if (gtid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNCW);
    }
    mbar_init(xbar, 1);
    mbar_fence_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmXS);
    tma_prefetch_desc(&tmW);
  }
  if (tid < 64) s_exp2[tid] = exp2((double)tid / 64.0);
  __syncthreads();

  // producer (thread 0 of the group): walks (unit, row tile, chunk) in consumption order
  int issued = 0;
  int pu = vb, prt = 0, pc = 0, pI = 0, pJ = 0, pnrt = 0, pnch = 0;
  if (pu < p.nunits) unit_dims(pu, pI, pJ, pnrt, pnch);
  auto pump = [&](int done) {
    if (gtid != 0) return;
    while (issued < total && issued < done + (S > 2 ? S - 1 : S)) {
      const int s = issued % S;
      if (issued >= S) mbar_wait(&empty[s], ((issued / S) & 1) ^ 1);
      unsigned char* XSs = stages + s * STAGE;
      unsigned char* Ws = XSs + nD * 2048;
      const int col0 = pJ * kSB + 16 * pc;
      mbar_arrive_expect_tx(&full[s], nD * 2048 + 1024);
      for (int dc = 0; dc < nD; ++dc) tma_load_2d(XSs + dc * 2048, &tmXS, 16 * dc, col0, &full[s]);
      tma_load_2d(Ws, &tmW, col0, 0, &full[s]);
      ++issued;
      if (++pc == pnch) {
        pc = 0;
        if (++prt == pnrt) {
          prt = 0;
          pu += vgrid;
          if (pu < p.nunits) unit_dims(pu, pI, pJ, pnrt, pnch);
        }
      }
    }
  };
  pump(0);

  const int g = lane >> 2, t = lane & 3;
  const int pg = perm8(g);
  int arow[2];
#pragma unroll
  for (int fr = 0; fr < 2; ++fr) arow[fr] = warp * 16 + 8 * fr + pg;
  uint32_t foff[4], foffs[4];
  const int sg = (g >> 1) + 4 * (g & 1);  // perm8^{-1}(g): C column 2t+v of fragment j is 8j+4v+t
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    foff[s] = swz_off(pg, 4 * s + t);
    foffs[s] = swz_off(sg, 4 * s + t);
  }
  const uint32_t a_base = (uint32_t)(warp * 16) * 128u;
  const double escale = p.escale;
  const bool l1 = p.kind == kL1;
  double* mycol = colacc + warp * kSB;
  int cons = 0, tiles_done = 0;

#pragma unroll 1
  for (int u = vb; u < p.nunits; u += vgrid) {
    int I, J, nrt, nch;
    unit_dims(u, I, J, nrt, nch);
    const bool offdiag = I != J;
    for (int i = lane; i < kSB; i += 32) mycol[i] = 0.0;
#pragma unroll 1
    for (int rt = 0; rt < nrt; ++rt) {
      const int64_t row0 = (int64_t)I * kSB + rt * 64;
      if (gtid == 0) {
        mbar_arrive_expect_tx(xbar, nD * 64 * 128);
        for (int dc = 0; dc < nD; ++dc) tma_load_2d(xt + dc * 64 * 128, &tmX, 16 * dc, (int)row0, xbar);
      }
      double sqr[2], gid[2], vrow[2], racc[2] = {0.0, 0.0};
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        const int64_t grow = row0 + arow[fr];
        const bool rin = grow < p.n;
        sqr[fr] = rin ? p.sqn[grow] : 0.0;
        gid[fr] = (double)grow;
        vrow[fr] = rin ? p.v[grow] : 0.0;
      }
      mbar_wait(xbar, tiles_done & 1);
      ++tiles_done;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        const int s = cons % S;
        mbar_wait(&full[s], (cons / S) & 1);
        __syncwarp();
        const unsigned char* XSs = stages + s * STAGE;
        const unsigned char* Ws = XSs + nD * 2048;
        const int col0 = J * kSB + 16 * c;
        double gv[2][2][2];
        if constexpr (GRAM) {
          double sqc4[2][2], idc4[2][2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int64_t col = col0 + 8 * j + 4 * v + t;
              const bool cin = col < p.n;
              sqc4[j][v] = cin ? __ldg(p.rec + col * p.prec + 1) : 0.0;
              idc4[j][v] = cin ? (double)col : -1.0;
            }
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j) gv[fr][j][0] = gv[fr][j][1] = 0.0;
#pragma unroll 1
          for (int dc = 0; dc < nD; ++dc) {
            const unsigned char* Xw = xt + dc * 64 * 128 + a_base;
            const unsigned char* Sw = XSs + dc * 2048;
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              double a[2];
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) a[fr] = *reinterpret_cast<const double*>(Xw + fr * 1024 + foff[s4]);
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const double bv = *reinterpret_cast<const double*>(Sw + j * 1024 + foffs[s4]);
#pragma unroll
                for (int fr = 0; fr < 2; ++fr) dmma884(gv[fr][j][0], gv[fr][j][1], a[fr], bv);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v)
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) {
                double dd = __dadd_rn(__dadd_rn(-2.0 * gv[fr][j][v], sqr[fr]), sqc4[j][v]);
                dd = clamp_pin(dd, gid[fr], idc4[j][v]);
                gv[fr][j][v] = kfun_eval(dd, p.kfun, escale, s_exp2);
              }
        } else {
          double dsum[2][2][2];
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j) dsum[fr][j][0] = dsum[fr][j][1] = 0.0;
#pragma unroll 1
          for (int dc = 0; dc < nD; ++dc) {
            const unsigned char* Xw = xt + dc * 64 * 128;
            const unsigned char* Sw = XSs + dc * 2048;
            const int jn = min(16, p.d - 16 * dc);
#pragma unroll 2
            for (int jj = 0; jj < jn; ++jj) {
              double xr[2], xs[2][2];
#pragma unroll
              for (int fr = 0; fr < 2; ++fr) xr[fr] = *reinterpret_cast<const double*>(Xw + swz_off(arow[fr], jj));
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                  xs[j][v] = *reinterpret_cast<const double*>(Sw + swz_off(8 * j + 4 * v + t, jj));
#pragma unroll
              for (int fr = 0; fr < 2; ++fr)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                  for (int v = 0; v < 2; ++v) {
                    const double df = __dsub_rn(xr[fr], xs[j][v]);
                    dsum[fr][j][v] = l1 ? __dadd_rn(dsum[fr][j][v], fabs(df))
                                        : __dadd_rn(dsum[fr][j][v], __dmul_rn(df, df));
                  }
            }
          }
#pragma unroll
          for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int v = 0; v < 2; ++v) gv[fr][j][v] = kfun_eval(dsum[fr][j][v], p.kfun, escale, s_exp2);
        }
        // row product: racc += A(R, chunk) v(chunk);  column product: A(R, chunk)^T v(R)
        double wv[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int v = 0; v < 2; ++v) wv[j][v] = *reinterpret_cast<const double*>(Ws + swz_off(0, 8 * j + 4 * v + t));
#pragma unroll
        for (int fr = 0; fr < 2; ++fr)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) racc[fr] = fma(gv[fr][j][v], wv[j][v], racc[fr]);
        if (offdiag) {
          double cp[2][2];
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              double x = fma(gv[1][j][v], vrow[1], gv[0][j][v] * vrow[0]);
              x += __shfl_xor_sync(0xffffffffu, x, 4);   // over the 8 row groups g (fixed tree)
              x += __shfl_xor_sync(0xffffffffu, x, 8);
              x += __shfl_xor_sync(0xffffffffu, x, 16);
              cp[j][v] = x;
            }
          if (lane < 4) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int v = 0; v < 2; ++v) mycol[16 * c + 8 * j + 4 * v + t] += cp[j][v];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++cons;
        if (warp == 0) pump(cons);
      }
      // this row tile's part of A(I, J) v(J): reduce over the quad, rows at arow
#pragma unroll
      for (int fr = 0; fr < 2; ++fr) {
        double r = racc[fr];
        r += __shfl_xor_sync(0xffffffffu, r, 1);
        r += __shfl_xor_sync(0xffffffffu, r, 2);
        const int64_t grow = row0 + arow[fr];
        if (t == 0 && grow < p.n) p.rowpart[(int64_t)u * kSB + rt * 64 + arow[fr]] = r;
      }
      gsync();  // the next row tile's X load overwrites xt
    }
    if (offdiag) {  // A(I, J)^T v(I): the four warps' slots in warp order
      for (int i = gtid; i < kSB; i += kGT) {
        double s2 = 0.0;
        for (int w = 0; w < kNCW; ++w) s2 += colacc[w * kSB + i];
        p.colpart[(int64_t)u * kSB + i] = s2;
      }
    }
    gsync();  // colacc is zeroed by the next unit
  }
}

// out[i] = sum_{J <= I} rowpart(I, J)[r] + sum_{I' > I} colpart(I', I)[r] + add, in block order
__global__ void symv_reduce_kernel(const double* __restrict__ rowpart,
                                   const double* __restrict__ colpart, int64_t n, int nsb,
                                   const double* __restrict__ add_vec, double add_coef,
                                   double add_const, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int I = (int)(i / kSB), r = (int)(i % kSB);
  double s = 0.0;
  for (int J = 0; J <= I; ++J) s += rowpart[((int64_t)I * (I + 1) / 2 + J) * kSB + r];
  for (int I2 = I + 1; I2 < nsb; ++I2) s += colpart[((int64_t)I2 * (I2 + 1) / 2 + I) * kSB + r];
  out[i] = s + (add_vec ? add_coef * add_vec[i] : 0.0) + add_const;
}

}  // namespace

int64_t symv_scratch_doubles(int64_t n) {
  const int64_t nsb = (n + kSB - 1) / kSB;
  return 2 * (nsb * (nsb + 1) / 2) * kSB;
}

// Returns false when this configuration does not fit (the caller uses the generic product).
bool launch_symv(const double* X, int64_t dpad, int d, const double* sqn, const double* rec,
                 int64_t prec, const double* v, int64_t ldv, int64_t n, int kind, int kfun,
                 double escale, double* scratch, const double* add_vec, double add_coef,
                 double add_const, double* out, cudaStream_t st) {
  constexpr int kMaxSmem = 227 * 1024;
  // below ~16 super-blocks the 1024-point units are too few to fill 148 SMs (n = 5000:
  // 1.9 ms against the generic product's 0.54 ms; n = 20000: 5.0 vs 9.2 ms)
  if (n < 16 * (int64_t)kSB) return false;
  const int nD = (int)(dpad / 16);
  int S = 4;
  while (S >= 2 && smem_bytes(S, nD) > kMaxSmem) --S;
  if (S < 2) return false;
  SymvParams p{};
  p.X = X;
  p.dpad = dpad;
  p.dchunks = nD;
  p.d = d;
  p.sqn = sqn;
  p.rec = rec;
  p.prec = prec;
  p.v = v;
  p.n = n;
  p.kind = kind;
  p.kfun = kfun;
  p.escale = escale;
  p.nsb = (int)((n + kSB - 1) / kSB);
  p.nunits = p.nsb * (p.nsb + 1) / 2;
  p.rowpart = scratch;
  p.colpart = scratch + (int64_t)p.nunits * kSB;
  CUtensorMap mX, mXS, mW;
  if (!(make_map(&mX, X, dpad, n, dpad, 64) && make_map(&mXS, rec + 2, dpad, n, prec, 16) &&
        make_map(&mW, v, n, 1, ldv, 8)))
    return false;
  const bool gram = kind == kGaussGram;
  const void* kfn = gram ? (const void*)symv_kernel<true> : (const void*)symv_kernel<false>;
  const int smem = smem_bytes(S, nD);
  if (ensure_smem_attr(kfn, kMaxSmem) != cudaSuccess) return false;
  const int occ = cached_occupancy(kfn, 256, smem, 1);
  const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)p.nunits + kG - 1) / kG,
                                                    (int64_t)occ * num_sms());
  if (gram) symv_kernel<true><<<grid, 256, smem, st>>>(p, S, mX, mXS, mW);
  else symv_kernel<false><<<grid, 256, smem, st>>>(p, S, mX, mXS, mW);
  symv_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p.rowpart, p.colpart, n, p.nsb,
                                                                   add_vec, add_coef, add_const,
                                                                   out);
  return true;
}

}  // namespace rpcb
